"""Q~v and Q~^T g of one step on two CUDA streams (independent operands) vs one stream:
device time per step on config 2 (or argv[1])."""
import sys

import torch

sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
pos, off = make_config(cfg, seed=1000)
N, m = int(off[-1]), len(off) - 1
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
v = torch.randn(3 * N, dtype=torch.float64, device="cuda")
g = torch.randn(3 * N - 6 * m, dtype=torch.float64, device="cuda")
main = torch.cuda.current_stream()
s2 = torch.cuda.Stream()


def one():
    op.apply("qtilde_v", v)
    op.apply("qtilde_tv", g)


def two():
    s2.wait_stream(main)
    with torch.cuda.stream(s2):
        op.apply("qtilde_tv", g)
    op.apply("qtilde_v", v)
    main.wait_stream(s2)


for name, f in (("one stream", one), ("two streams", two), ("one stream", one), ("two streams", two)):
    for _ in range(5):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(100):
        f()
    b.record()
    torch.cuda.synchronize()
    print(f"cfg{cfg} {name}: {a.elapsed_time(b) / 100:.4f} ms per step")
