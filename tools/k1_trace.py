"""K1 MMA-issuer time split (needs a -DQJL_K1_TRACE=1 library via QJL_LIB): per CTA, cycles
waiting for the tile's A operand (at_full), for an accumulator buffer (t_empty), for S_full
(b_full), and the rest (issuing), over one C4 prefill K1 launch."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2406_03482_b200 import _lib
from paper_2406_03482_b200.distributed import shard_units

r = bench.measure_prefill(torch.device("cuda", 0), 0, lambda t: shard_units(t, 1, 0), steps=3, warmup=1, parity=False)
lib = _lib.load()
buf = np.zeros((148, 6), dtype=np.uint64)
lib.qjl_debug_k1_trace.restype = ctypes.c_int
lib.qjl_debug_k1_trace(buf.ctypes.data_as(ctypes.c_void_p), 148)
tot = buf[:, 4].astype(float)
print("K1 kernel_ms", round(r["kernel_ms"] * 1e3, 1), "us; tiles/CTA", buf[:, 5].mean())
for i, name in enumerate(["wait A (at_full)", "wait accumulator (t_empty)", "wait S_full (b_full)", "issue + other"]):
    f = buf[:, i].astype(float) / tot
    print(f"{name:28s} mean {f.mean():.3f}  min {f.min():.3f}  max {f.max():.3f}")
print("cycles per tile (mean)", (tot / buf[:, 5].astype(float)).mean())
