import sys, time
import torch
sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq
from paper_1708_08427_b200.workloads import make_config
cfg = int(sys.argv[1])
pos, off = make_config(cfg, seed=1000)
model = rq.MultiBodyModel.from_arrays(pos, off)
for i in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op = rq.MultiBodyOperator(model)
    torch.cuda.synchronize()
    print(f"cfg{cfg} setup {i}: {time.perf_counter() - t0:.3f} s", flush=True)
    del op
