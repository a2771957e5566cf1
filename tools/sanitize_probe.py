"""Small-shape run of every tensor-core kernel for compute-sanitizer (memcheck / racecheck /
synccheck): fused prompt profile (k_detect_partial, k_detect_finish_build), K1 (k_quant_tc),
P2T value quantizer, query-sketch prep (k_uprep, with and without the decode-step append),
k_udecode (stream-K, deterministic, chained), k_uscores and the chained benchmark hook."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2406_03482_b200.device import DeviceKeyCache

torch.manual_seed(0)
U, n, G, d = 4, 600, 4, 128
K = (torch.randn(U, n + 4, d, device="cuda") * torch.exp(torch.randn(U, 1, d, device="cuda"))).bfloat16()
V = torch.randn(U, n + 4, d, device="cuda").bfloat16()
q = torch.randn(U, G, d, device="cuda").bfloat16()
c = DeviceKeyCache.create(U, d, 256, h=8, m_out=64, capacity=n + 128, seed=1)
c.prefill(K[:, :n], V[:, :n])                       # profile + S_full, K1, value quantizer
out = c.decode(q)
out2 = c.decode(q, chained=True)
out3 = c.decode(q, deterministic=True)
lg = c.scores(q)
for i in range(3):                                  # decode steps with the fused append
    c.decode_step(q, K[:, n + i], V[:, n + i], chained=i > 0)
ms = c.bench_decode_kernel(q, reps=2)
torch.cuda.synchronize()
assert torch.isfinite(out).all() and torch.allclose(out, out2, rtol=1e-4, atol=1e-6) and torch.isfinite(lg).all()
print("sanitize probe ok", float(out.abs().sum()), float(out3.abs().sum()), ms)
