"""Probe: the scan kernel reading the queries straight from page-locked host
memory (UVA; the kernel's cp.async staging goes over PCIe) vs the copy engine.
c2-like shapes; medians of CUDA-event times (ms)."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1509_05186_b200 import api  # noqa: E402
from paper_1509_05186_b200._lib import check  # noqa: E402


def timeit(fn, n=15, flush=None):
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    fn()
    torch.cuda.synchronize()
    for a, b in evs:
        if flush is not None:
            flush.fill_(1.0)
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return sorted(a.elapsed_time(b) for a, b in evs)[n // 2]


def main():
    Q, d, k = 10_000, 128, 100
    rng = np.random.default_rng(0)
    cb = rng.uniform(0, 255, (8, 256, 16)).astype(np.float32)
    distinct = rng.integers(0, 256, (600, 8), dtype=np.uint8)
    codes = distinct[rng.integers(0, 600, 1_000_000)]
    qx = rng.uniform(0, 255, (Q, d)).astype(np.float32)
    ix = api.Index.et_build_etree(codes)
    cbd = torch.from_numpy(cb).cuda()
    qh = torch.from_numpy(qx).pin_memory()
    qd = qh.cuda()
    rd = torch.empty(Q, k, device="cuda")
    ri = torch.empty(Q, k, dtype=torch.int32, device="cuda")
    dh = torch.empty(Q, k).pin_memory()
    ih = torch.empty(Q, k, dtype=torch.int32).pin_memory()
    flush = torch.empty(512 << 18, device="cuda")
    ws = ix._workspace(ix.et_workspace_size(Q, k), qd.device)
    lib = api._lib.load()
    st = torch.cuda.current_stream().cuda_stream

    def step(qptr):
        check(lib.et_etree_topk(ix._h, cbd.data_ptr(), d, None, qptr, Q, k, rd.data_ptr(), ri.data_ptr(),
                                ws.data_ptr(), ws.numel(), st))
    step(qd.data_ptr())
    torch.cuda.synchronize()
    ref = (rd.clone(), ri.clone())
    step(qh.data_ptr())
    torch.cuda.synchronize()
    print("zero-copy results equal:", torch.equal(rd, ref[0]) and torch.equal(ri, ref[1]))
    for rep in range(2):
        print("device step", timeit(lambda: step(qd.data_ptr()), flush=flush),
              "| zero-copy step", timeit(lambda: step(qh.data_ptr()), flush=flush),
              "| h2d", timeit(lambda: qd.copy_(qh, non_blocking=True), flush=flush),
              "| serial e2e", timeit(lambda: (qd.copy_(qh, non_blocking=True), step(qd.data_ptr()),
                                             dh.copy_(rd, non_blocking=True), ih.copy_(ri, non_blocking=True)),
                                     flush=flush),
              "| zero-copy e2e", timeit(lambda: (step(qh.data_ptr()), dh.copy_(rd, non_blocking=True),
                                                ih.copy_(ri, non_blocking=True)), flush=flush),
              "| host call", timeit(lambda: ix.et_etree_topk_host(k, qh, cbd, out=(dh, ih)), flush=flush))


if __name__ == "__main__":
    main()
