"""HBM bandwidth probes on the B200 (CUDA events, best of N): read-only
(torch reductions over 4 GiB), read+write (copy_, the MEASURED_PEAKS form),
write-only (fill_).  Context for the roofline fractions: K1 only reads, K2
reads ~3.6x what it writes.

    python tools/read_bw.py
"""
import json

import torch


def best_ms(fn, reps=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    n = 1 << 30  # 4 GiB of fp32
    a = torch.empty(n, dtype=torch.float32, device="cuda").uniform_()
    b = torch.empty_like(a)
    out = {}
    out["read_sum_gbs"] = n * 4 / (best_ms(lambda: a.sum()) * 1e-3) / 1e9
    out["read_amax_gbs"] = n * 4 / (best_ms(lambda: torch.amax(a)) * 1e-3) / 1e9
    out["copy_rw_gbs"] = 2 * n * 4 / (best_ms(lambda: b.copy_(a)) * 1e-3) / 1e9
    out["write_fill_gbs"] = n * 4 / (best_ms(lambda: b.fill_(1.0)) * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
