"""Run only the config-4 prefill (K1) measurement of bench.py (for ncu / A-B)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
from paper_2406_03482_b200.distributed import shard_units
print(json.dumps(bench.measure_prefill(torch.device("cuda", 0), 0, lambda total: shard_units(total, 1, 0),
                                       steps=steps, warmup=2), default=bench._jsonable))
