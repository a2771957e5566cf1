"""Run the C4 prefill pipeline (fused profile + K1) a few times, for ncu launch lists."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2406_03482_b200.device import DeviceKeyCache

U, n, d = 128, 8192, 128
g = torch.Generator(device="cuda").manual_seed(0)
K = (torch.randn(U, n, d, generator=g, device="cuda") *
     torch.exp(torch.randn(U, 1, d, generator=g, device="cuda"))).to(torch.bfloat16)
c = DeviceKeyCache.create(U, d, 512, h=8, m_out=64, capacity=n, key_dtype=torch.bfloat16, with_values=False)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    c.n = 0
    c.prefill(K)
torch.cuda.synchronize()
print("ok")
