"""Per-CTA phase durations of the scan kernel (experiment build with -DET_PHASE_TIMING).

  python tools/phase_timing.py --config c2
Phases: 0 start, 1 build start, 5 staged, 6 round 0 built (levels 0-3), 7 TMEM levels copied,
2 build done, 3 scan done, 4 compaction done.  s = 60 joined forests (c3): 1 setup done,
5/6 tree 1 tables/scan, 7/2 tree 0 tables/scan, 3 join done, 4 end.
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.environ.get("ET_PHASE_LIB") or os.path.join(ROOT, "paper_1509_05186_b200", "_build", "phase", "libetree.so")
os.environ["ET_LIB_PATH"] = LIB

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    import torch
    from paper_1509_05186_b200 import api
    from paper_1509_05186_b200 import synth
    cfg = synth.CONFIGS[a.config]
    dev = torch.device("cuda", 0)
    st = bench.prepare(cfg, {}, bench.CudaBackend(dev), bench.Comm(0, 1), "none")
    ix = bench.build_index(cfg, st)
    st["q_dev"] = torch.from_numpy(st["qx"]).to(dev)
    st["cb_dev"] = torch.from_numpy(st["cb"]).to(dev)
    for _ in range(3):
        if cfg.ivf_nlist:   # IVF (c4): the same scan kernel over (cell, queries) chunks
            ix.et_ivf_topk(st["q_dev"], nprobe=cfg.ivf_nprobe, k=cfg.topk)
        else:
            ix.et_etree_topk(cfg.topk, queries=st["q_dev"], codebooks=st["cb_dev"])
    torch.cuda.synchronize()
    lib = api._lib.load()
    n = 1 << 16
    buf = np.zeros((n, 8), dtype=np.uint64)
    s60 = cfg.d // cfg.M == 60
    fn = lib.et_debug_phases_s60 if s60 else lib.et_debug_phases
    fn.argtypes = [C.c_void_p, C.c_int]
    fn(buf.ctypes.data, n)
    used = buf[:, 0] > 0
    b = buf[used].astype(np.float64)
    t0 = b[:, 0].min()
    order = [(0, 1, "start->build"), (1, 5, "stage"), (5, 6, "round 0"), (6, 7, "TMEM copy"),
             (7, 2, "round 1"), (2, 3, "scan"), (3, 4, "compaction")]
    if s60 and b[:, 6].max() > 0:   # joined forest (T = 2): tree 1 tables/scan, tree 0 tables/scan, join
        order = [(0, 1, "setup"), (1, 5, "tables tree 1"), (5, 6, "scan tree 1"), (6, 7, "tables tree 0"),
                 (7, 2, "scan tree 0"), (2, 3, "join"), (3, 4, "tail")]
    elif s60:   # narrow forest scan (narrow_kernel): staging, 16 levels' tables, tuple scan
        order = [(0, 1, "stage"), (1, 5, "tables (16 levels)"), (5, 3, "tuple scan"), (3, 4, "tail")]
    print(f"units {used.sum()}  kernel span {(b[:, 4].max() - t0) / 1e3:.1f} us")
    for i, j, name in order:
        d = (b[:, j] - b[:, i]) / 1e3
        print(f"{name:14s} mean {d.mean():7.2f} us  p50 {np.median(d):7.2f}  max {d.max():7.2f}")
    tot = (b[:, 4] - b[:, 0]) / 1e3
    print(f"{'total/CTA':14s} mean {tot.mean():7.2f} us")


if __name__ == "__main__":
    main()
