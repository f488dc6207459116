"""Vendor reference point (NOT the product path): cuFFT fp64 via torch.fft on the
shapes of the 512^3 padded pipeline.  Reports ms and effective GB/s (read+write)."""
import json
import torch

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps

n = 512; m = 768; k = n // 2 + 1
out = {}
x = torch.randn(2 * 3 * m * m, m, dtype=torch.float64, device="cuda")  # 6 real z-pencils per (x,y)... 2 reps of 3
ms = t(lambda: torch.fft.rfft(x, dim=1))
out["rfft_z_768_batch"] = dict(ms=ms, GBps=(x.numel() * 8 + x.shape[0] * (m // 2 + 1) * 16) / ms / 1e6)
del x
c = torch.randn(6 * m, n, k, dtype=torch.complex128, device="cuda")
ms = t(lambda: torch.fft.fft(c, dim=1))
out["c2c_y_512_strided(6*768,512,257)"] = dict(ms=ms, GBps=2 * c.numel() * 16 / ms / 1e6)
del c
c = torch.randn(6 * m * m, m, dtype=torch.complex128, device="cuda")
ms = t(lambda: torch.fft.fft(c, dim=1))
out["c2c_contig_768(6*768^2)"] = dict(ms=ms, GBps=2 * c.numel() * 16 / ms / 1e6)
del c
# padded pipeline reference: irfftn of (6, 768, 768, 385) + rfftn of (3, 768,768,768)
s = torch.randn(6, m, m, m // 2 + 1, dtype=torch.complex128, device="cuda")
ms_i = t(lambda: torch.fft.irfftn(s, s=(m, m, m), dim=(1, 2, 3)), reps=2)
del s
r = torch.randn(3, m, m, m, dtype=torch.float64, device="cuda")
ms_f = t(lambda: torch.fft.rfftn(r, dim=(1, 2, 3)), reps=2)
out["cufft_padded_irfftn6+rfftn3_ms"] = ms_i + ms_f
print(json.dumps(out))
