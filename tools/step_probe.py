"""Generation-step timing at C3 (row F1): append one token's key and value per unit,
then decode over the grown cache -- against the decode alone.  CUDA events, inputs on
the device."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench

w = dict(bench.WORKLOADS["c3"])
dev = torch.device("cuda", 0)
cache = bench.build_cache(w, 0, 0, dev)
cache.n = cache.n_values = 32768 - 128   # leave room for the appended tokens
U, d, G = w["batch"] * w["kv_heads"], w["d"], w["G"]
cap_n = cache.n
q = torch.randn(U, G, d, device=dev).to(torch.bfloat16)
kn = torch.randn(U, 1, d, device=dev).to(torch.bfloat16)
vn = torch.randn(U, 1, d, device=dev).to(torch.bfloat16)
out = torch.empty(U, G, d, device=dev)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
res = {}
for mode in ("decode", "append_k", "append_kv", "step", "decode_step"):
    for rep in range(2):
        steps = 100
        torch.cuda.synchronize()
        e0.record()
        for i in range(steps):
            if mode == "decode_step":
                cache.n = cache.n_values = cap_n + (i % 100)
                cache.decode_step(q, kn[:, 0], vn[:, 0], out=out)
                continue
            if mode != "decode":
                cache.n = cache.n_values = cap_n + (i % 100)
                cache.append_keys(kn)
                if mode in ("append_kv", "step"):
                    cache.append_values(vn)
            if mode in ("decode", "step"):
                cache.decode(q, out=out)
        e1.record()
        torch.cuda.synchronize()
        res[mode] = e0.elapsed_time(e1) / steps * 1e3
    cache.n = cache.n_values = cap_n
print(json.dumps({k: round(v, 2) for k, v in res.items()}), "us per call")
