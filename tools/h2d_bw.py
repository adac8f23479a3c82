"""Host-to-device bandwidth from pinned memory (CUDA events, best of N): one
copy vs the same bytes split over 2 / 4 streams -- the e2e ceiling context.

    python tools/h2d_bw.py
"""
import json

import torch


def main():
    n = 378_702_080  # one config-B step of e2e inputs
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(4)]
    out = {}
    for k in (1, 2, 4):
        best = 1e30
        for _ in range(6):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream()
            e0.record(cur)
            step = n // k
            for i in range(k):
                s = streams[i]
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    d[i * step:(i + 1) * step if i + 1 < k else n].copy_(
                        h[i * step:(i + 1) * step if i + 1 < k else n], non_blocking=True)
                cur.wait_stream(s)
            e1.record(cur)
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"h2d_gbs_{k}_streams"] = n / (best * 1e-3) / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()
