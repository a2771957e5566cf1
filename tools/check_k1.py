"""Quick check: tensor-core K1 vs the generic fp64 SIMT K1 on the same inputs."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2406_03482_b200.device import DeviceKeyCache

def run(U, n, m_in, h, m_out, dt, force_simt):
    if force_simt: os.environ["QJL_FORCE_SIMT"] = "1"
    g = torch.Generator(device="cuda"); g.manual_seed(5)
    K = (torch.randn(U, n, 128, generator=g, device="cuda") * torch.exp(torch.randn(U, 1, 128, generator=g, device="cuda"))).to(dt)
    c = DeviceKeyCache.create(U, 128, m_in, h=h, m_out=m_out, capacity=n, seed=1, key_dtype=dt, with_values=False)
    if h: c.detect_outliers(K); c.set_sketches(c.S_in_host, c.S_out_host)
    torch.cuda.synchronize(); t0 = time.time()
    c.append_keys(K); torch.cuda.synchronize(); t = time.time() - t0
    os.environ.pop("QJL_FORCE_SIMT", None)
    return c, t

for (U, n, m_in, h, m_out, dt) in [(2, 300, 256, 0, 0, torch.bfloat16), (4, 1000, 256, 8, 64, torch.bfloat16),
                                    (3, 700, 256, 4, 128, torch.float16), (4, 2048, 512, 8, 64, torch.bfloat16)]:
    a, ta = run(U, n, m_in, h, m_out, dt, False)
    b, tb = run(U, n, m_in, h, m_out, dt, True)
    db = (a.bits_in[:, :n] != b.bits_in[:, :n]).sum().item()
    dbo = (a.bits_out[:, :n] != b.bits_out[:, :n]).sum().item() if a.bits_out is not None else 0
    dn = (a.norm_in[:, :n] != b.norm_in[:, :n]).sum().item()
    dno = (a.norm_out[:, :n] != b.norm_out[:, :n]).sum().item() if a.norm_out is not None else 0
    print(f"U={U} n={n} m_in={m_in} h={h} {dt}: bytes differing in={db} out={dbo} norms in={dn} out={dno}  tc {ta*1e3:.1f} ms simt {tb*1e3:.1f} ms", flush=True)
