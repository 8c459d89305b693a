"""PCIe probe for the e2e bounds: pinned host <-> device copy bandwidth one
way, both ways at once, and in the byte mix of the e2e entries (16 B in /
10 B out per param for co2_outer_step_host; 4 B in / 2 B out for
co2_round_host in bf16-mixed).

  python tools/pcie_probe.py [--gib 1]
"""
import argparse
import time


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gib", type=float, default=1.0, help="bytes per transfer, GiB")
    a = ap.parse_args()
    import torch

    n = int(a.gib * (1 << 30))
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def t(f, reps=5):
        f()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            f()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    h2d = t(lambda: d.copy_(h, non_blocking=True))
    d2h = t(lambda: h.copy_(d, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)

    bi = t(both)
    print(f"H2D {n / h2d / 1e9:.1f} GB/s  D2H {n / d2h / 1e9:.1f} GB/s  "
          f"bidir {2 * n / bi / 1e9:.1f} GB/s total")
    for name, bin_, bout in (("co2_outer_step_host", 16, 10), ("co2_round_host", 4, 2)):
        m_in, m_out = int(n * bin_ / (bin_ + bout)), int(n * bout / (bin_ + bout))

        def mix():
            with torch.cuda.stream(s1):
                d[:m_in].copy_(h[:m_in], non_blocking=True)
            with torch.cuda.stream(s2):
                h2[:m_out].copy_(d2[:m_out], non_blocking=True)

        mt = t(mix)
        print(f"{name} mix ({bin_} B in / {bout} B out per param): {n / mt / 1e9:.1f} GB/s "
              f"combined -> {n / (bin_ + bout) / mt / 1e9:.2f}e9 params/s ceiling "
              "(both directions overlapped)")


if __name__ == "__main__":
    main()
