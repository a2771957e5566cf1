"""C3-shaped scores-only K2 (64 units x 32768 tokens, G = 4): times qjl_scores and runs it
a few times for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2406_03482_b200.distributed import shard_units

w = dict(bench.WORKLOADS["c3"])
if len(sys.argv) > 2:
    w["n"] = int(sys.argv[2])
sh = shard_units(64, 1, 0)
c = bench.build_cache(w, sh, 0, torch.device("cuda"))
q = bench.make_queries(w, sh, 0, torch.device("cuda"))
out = torch.empty(64, 4, c.n, device="cuda")
reps = 3 if len(sys.argv) > 1 and sys.argv[1] == "ncu" else 50
for _ in range(3):
    c.scores(q, out=out)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    c.scores(q, out=out, chained=True)
e1.record()
torch.cuda.synchronize()
print(f"scores: {e0.elapsed_time(e1) / reps * 1e3:.1f} us/step")
