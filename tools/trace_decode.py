"""One C3 decode with the QJL_UD_TRACE library: per-CTA globaltimer stamps (start, main
loop end, kernel end) -> timeline summary."""
import os, sys, subprocess, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
w = bench.WORKLOADS["c3"]
dev = torch.device("cuda", 0)
cache = bench.build_cache(w, 0, 0, dev)
q = torch.randn(64, 4, 128, device=dev).bfloat16()
for _ in range(3):
    cache.decode(q)
torch.cuda.synchronize()
print("MARK", flush=True)
cache.decode(q)
torch.cuda.synchronize()
