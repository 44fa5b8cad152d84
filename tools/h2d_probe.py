"""H2D copy-engine concurrency probe: 5.12 MB (c2 queries) as 1, 2, 4, 8
concurrent slices on separate streams; D2H 8 MB likewise.  Median ms."""
import torch


def timeit(fn, n=15):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    fn()
    torch.cuda.synchronize()
    for a, b in evs:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in evs)[n // 2]


def main():
    cur = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in range(8)]
    for nbytes, label in ((5_120_000, "h2d"), (8_000_000, "d2h")):
        h = torch.empty(nbytes // 4).pin_memory()
        h.fill_(1.0)
        dv = torch.empty(nbytes // 4, device="cuda")
        for ns in (1, 2, 4, 8):
            sl = [slice(i * len(h) // ns, (i + 1) * len(h) // ns) for i in range(ns)]

            def go():
                for s, x in zip(streams, sl):
                    s.wait_stream(cur)
                    with torch.cuda.stream(s):
                        if label == "h2d":
                            dv[x].copy_(h[x], non_blocking=True)
                        else:
                            h[x].copy_(dv[x], non_blocking=True)
                for s in streams[:ns]:
                    cur.wait_stream(s)
            t = timeit(go)
            print(f"{label} {nbytes/1e6:.2f} MB in {ns} streams: {t:.4f} ms = {nbytes / t / 1e6:.1f} GB/s")


if __name__ == "__main__":
    main()
