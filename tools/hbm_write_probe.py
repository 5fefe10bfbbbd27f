"""Write-dominated HBM ceiling on this B200 (for K7's roofline note): torch fill_ (write only) and a
1:12 read:write copy pattern (K7's per-prompt mix: 1 B class read, 12 B written), CUDA-event timed,
best of 10 after warm-up, 1 GiB+ buffers (larger than L2)."""
import json
import torch

dev = torch.device("cuda", 0)


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return best


out = {}
n = 1 << 28                                              # 1 GiB of int32
x = torch.empty(n, dtype=torch.int32, device=dev)
ms = t(lambda: x.fill_(7))
out["fill_int32_GBps"] = 4 * n / ms / 1e6
y = torch.empty(n, dtype=torch.int32, device=dev)
ms = t(lambda: y.copy_(x))
out["copy_int32_GBps_rw"] = 8 * n / ms / 1e6
# K7-like mix: 64M bytes read, 3 x 64M int32 written
m = 1 << 26
cls = torch.randint(0, 16, (m,), dtype=torch.uint8, device=dev)
o1 = torch.empty(m, dtype=torch.int32, device=dev)
o2 = torch.empty(m, dtype=torch.int32, device=dev)
o3 = torch.empty(m, dtype=torch.int32, device=dev)


def mix():
    c = cls.to(torch.int32)                              # extra temp: reads 64 MB, writes 256 MB
    o1.copy_(c)
    o2.copy_(c)
    o3.copy_(c)


ms = t(mix)
out["k7_mix_note"] = "cls->int32 temp + 3 copies: 64M x (1 + 4) + 3 x 64M x 8 bytes"
out["k7_mix_GBps"] = (m * 5 + 3 * m * 8) / ms / 1e6
print(json.dumps(out))
