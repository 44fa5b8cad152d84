"""Copy-engine probe for the e2e path (c2 shapes): H2D 5.12 MB of queries and
D2H 8 MB of results on the legacy stream vs side streams, concurrent, and the
host-buffer call (eager / graph) per batch count.  CUDA events, ms."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


FLUSH = None


def timeit(fn, n=10):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    fn()
    torch.cuda.synchronize()
    for a, b in evs:
        if FLUSH is not None:
            FLUSH.fill_(1.0)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in evs)[n // 2]


def main():
    Q, d, k = 10_000, 128, 100
    qh = torch.randn(Q, d).pin_memory()
    qd = torch.empty(Q, d, device="cuda")
    rd = torch.empty(Q, k, device="cuda")
    ri = torch.empty(Q, k, dtype=torch.int32, device="cuda")
    dh = torch.empty(Q, k).pin_memory()
    ih = torch.empty(Q, k, dtype=torch.int32).pin_memory()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    cur = torch.cuda.current_stream()
    print("h2d legacy", timeit(lambda: qd.copy_(qh, non_blocking=True)))
    print("d2h legacy", timeit(lambda: (dh.copy_(rd, non_blocking=True), ih.copy_(ri, non_blocking=True))))

    def side(fn, s):
        s.wait_stream(cur)
        with torch.cuda.stream(s):
            fn()
        cur.wait_stream(s)
    print("h2d side", timeit(lambda: side(lambda: qd.copy_(qh, non_blocking=True), s1)))
    print("d2h side", timeit(lambda: side(lambda: (dh.copy_(rd, non_blocking=True), ih.copy_(ri, non_blocking=True)), s2)))

    def both():
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            qd.copy_(qh, non_blocking=True)
        with torch.cuda.stream(s2):
            dh.copy_(rd, non_blocking=True)
            ih.copy_(ri, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)
    print("h2d || d2h", timeit(both))

    from paper_1509_05186_b200 import api
    rng = np.random.default_rng(0)
    cb = rng.uniform(0, 255, (8, 256, 16)).astype(np.float32)
    distinct = rng.integers(0, 256, (600, 8), dtype=np.uint8)
    codes = distinct[rng.integers(0, 600, 1_000_000)]
    qx = rng.uniform(0, 255, (Q, d)).astype(np.float32)
    ix = api.Index.et_build_etree(codes)
    cbd = torch.from_numpy(cb).cuda()
    qh2 = torch.from_numpy(qx).pin_memory()
    qd2 = qh2.cuda()
    print("device step", timeit(lambda: ix.et_etree_topk(k, queries=qd2, codebooks=cbd, out=(rd, ri))))
    global FLUSH
    for rep in range(2):
        FLUSH = None if rep == 0 else torch.empty(512 << 18, device="cuda")
        print(f"flush={rep}: h2d", timeit(lambda: qd.copy_(qh2, non_blocking=True)),
              "d2h", timeit(lambda: (dh.copy_(rd, non_blocking=True), ih.copy_(ri, non_blocking=True))),
              "serial", timeit(lambda: (qd.copy_(qh2, non_blocking=True),
                                         ix.et_etree_topk(k, queries=qd, codebooks=cbd, out=(rd, ri)),
                                         dh.copy_(rd, non_blocking=True), ih.copy_(ri, non_blocking=True))))
    for nb in (1, 2, 4, 8):
        for eager in (0, 1):
            if eager:
                os.environ["ET_HOST_EAGER"] = "1"
            else:
                os.environ.pop("ET_HOST_EAGER", None)
            print(f"host call nb={nb} eager={eager}",
                  timeit(lambda: ix.et_etree_topk_host(k, qh2, cbd, out=(dh, ih), n_batches=nb)))


if __name__ == "__main__":
    main()
