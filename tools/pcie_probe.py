import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True); h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda"); d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f, reps=5):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps
h2d = t(lambda: d.copy_(h, non_blocking=True)); d2h = t(lambda: h.copy_(d, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
bi = t(both)
print(f"H2D {n/h2d/1e9:.1f} GB/s  D2H {n/d2h/1e9:.1f} GB/s  bidir {2*n/bi/1e9:.1f} GB/s total")
# the e2e mix: 16 B in, 10 B out per param
m_in, m_out = int(n * 16 / 26), int(n * 10 / 26)
def mix():
    with torch.cuda.stream(s1): d[:m_in].copy_(h[:m_in], non_blocking=True)
    with torch.cuda.stream(s2): h2[:m_out].copy_(d2[:m_out], non_blocking=True)
mt = t(mix)
print(f"26 B/param mix: {n/mt/1e9:.1f} GB/s combined -> {n/26/mt/1e9:.2f}e9 params/s ceiling")
