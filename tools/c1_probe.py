"""Config-1 leg of bench.py alone (fp32 keys -> fp64 quantizer + K2 logits), for A/B runs."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
r = bench.measure_c1(torch.device("cuda", 0), 0)
print(json.dumps({k: r[k] for k in ("k1_ms", "keys_per_s", "scores_ms")} | {"pass": r["parity"]["pass"]}))
