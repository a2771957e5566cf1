"""Run only the config-4 prefill (K1) measurement of bench.py (for ncu / A-B)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
print(json.dumps(bench.measure_prefill(torch.device("cuda", 0), 0, steps=steps, warmup=2)))
