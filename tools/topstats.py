"""Print top-tree statistics of the config-2 plan (set RQ_VERBOSE=1, RQ_TILE_HEIGHT=H)."""
import sys

sys.path.insert(0, ".")
import paper_1708_08427_b200 as rq  # noqa: E402
from paper_1708_08427_b200.workloads import make_config  # noqa: E402

pos, off = make_config(int(sys.argv[1]) if len(sys.argv) > 1 else 2, seed=1000)
op = rq.MultiBodyOperator(rq.MultiBodyModel.from_arrays(pos, off))
info = op.plan.info()
print({k: info[k] for k in ("chunk_smem", "chunk_ctas_per_sm", "chunk_smem_bytes", "n_chunks")})
