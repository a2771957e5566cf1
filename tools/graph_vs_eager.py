"""Eager chained decode steps vs the same steps replayed from a CUDA graph, alternated
(eager, graph, eager, graph) so a drift of the box shows up in both.
usage: python tools/graph_vs_eager.py BATCH N M_IN [STEPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2406_03482_b200.distributed import shard_units

batch, n, m_in = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 50
w = dict(bench.WORKLOADS["c5"], batch=batch, n=n, m_in=m_in)
dev = torch.device("cuda", 0)
U = w["batch"] * w["kv_heads"]
shard = shard_units(U, 1, 0)
cache = bench.build_cache(w, shard, 0, dev)
q = bench.make_queries(w, shard, 0, dev)
out = torch.empty(U, w["G"], w["d"], dtype=torch.float32, device=dev)
for i in range(5):
    cache.decode(q, out=out, chained=i > 0)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for i in range(steps):
        cache.decode(q, out=out, chained=i > 0)
g.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def eager():
    cache.decode(q, out=out)
    e0.record()
    for _ in range(steps):
        cache.decode(q, out=out, chained=True)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3


def graph():
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps * 1e3


for r in range(3):
    print(f"B{batch} n{n} m{m_in} round {r}: eager {eager():.1f} us/step, graph {graph():.1f} us/step", flush=True)
