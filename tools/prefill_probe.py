"""C4 prefill pipeline timing breakdown: fused profile alone, K1 alone, prefill (profile + K1),
device time (CUDA events) and host time per call; `ncu` mode just runs prefill a few times."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_03482_b200 import _lib
from paper_2406_03482_b200.device import _TORCH2QJL, DeviceKeyCache, _stream

U, n, d = 128, 8192, 128
g = torch.Generator(device="cuda").manual_seed(0)
K = (torch.randn(U, n, d, generator=g, device="cuda") *
     torch.exp(torch.randn(U, 1, d, generator=g, device="cuda"))).to(torch.bfloat16)
c = DeviceKeyCache.create(U, d, 512, h=8, m_out=64, capacity=n, key_dtype=torch.bfloat16, with_values=False)
if len(sys.argv) > 1 and sys.argv[1] == "ncu":
    for _ in range(3):
        c.n = 0
        c.prefill(K)
    torch.cuda.synchronize()
    sys.exit(0)
c.prefill(K)
sin, sout = c._sk_op
mags = torch.empty(U, d, dtype=torch.float64, device="cuda")
dws = c._detect_ws(n)


def profile():
    _lib.check(c.lib.qjl_prefill_profile(K.data_ptr(), _TORCH2QJL[K.dtype], U, n, d, n * d, 8, sin.data_ptr(),
                                         sout.data_ptr(), 512, 64, _TORCH2QJL[c.sketch_dtype], c.channels.data_ptr(),
                                         mags.data_ptr(), c.s_full.data_ptr(), dws.data_ptr(), dws.numel(),
                                         _stream()), "profile")


def k1():
    c.n = 0
    c.append_keys(K)


def both():
    c.n = 0
    c.prefill(K)


for name, fn in (("profile", profile), ("k1", k1), ("prefill", both)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    print(f"{name:8s} device {e0.elapsed_time(e1) / 20 * 1e3:8.1f} us/call, host {(t1 - t0) / 20 * 1e6:8.1f} us/call")
