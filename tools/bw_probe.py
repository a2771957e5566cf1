"""Read-bandwidth probe: torch reductions over buffers shaped like the C3 cache arrays."""
import torch
dev = "cuda"
def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
big = torch.randint(0, 255, (193 * 1024 * 1024 // 4,), dtype=torch.int32, device=dev)
ms = t(lambda: big.sum())
print(f"contiguous 193 MB int32 sum: {ms*1e3:.1f} us -> {big.numel()*4/ms/1e6:.0f} GB/s")
dst = torch.empty_like(big)
ms = t(lambda: dst.copy_(big))
print(f"contiguous 193 MB copy (r+w): {ms*1e3:.1f} us -> {2*big.numel()*4/ms/1e6:.0f} GB/s")
arrs = [torch.randint(0, 255, (64, 32768, nb // 4), dtype=torch.int32, device=dev) for nb in (32, 8, 32)] + \
       [torch.randint(0, 255, (64, 32768, 2), dtype=torch.int32, device=dev) for _ in range(2)] + \
       [torch.randint(0, 255, (64, 32768), dtype=torch.int16, device=dev) for _ in range(2)]
tot = sum(x.numel() * x.element_size() for x in arrs)
ms = t(lambda: [x.sum() for x in arrs])
print(f"7 cache-shaped arrays ({tot/1e6:.0f} MB), one sum each: {ms*1e3:.1f} us -> {tot/ms/1e6:.0f} GB/s")
