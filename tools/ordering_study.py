"""Encoding-ordering study (P:358-371 [§4.3]), synthetic rerun.

The paper builds the E-Tree over the original chunk order and over a shuffled
chunk order and reports that the order has "relatively small impact on the
number of postfix/prefix length".  This tool does the same on the
synthetic stand-ins: for each chunk order (original, reversed, a
few seeded shuffles) it builds the index with `byte_perm`, reads the tree
statistics (internal nodes L1, leaves L2, Σpostfix, lookups) from
`et_index_stats`, times the hot path (`et_etree_topk`, L2 flushed between
steps, CUDA events) and checks that the top-k distances do not depend on the
order (the permutation only reorders the summands' tree positions; the sum
order follows the permuted levels, so distances agree to fp32 rounding).

  python tools/ordering_study.py --configs c2 u1m c3 --out profiles/r02_ordering.md
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def orders(M, n_random, seed):
    out = [("original", np.arange(M, dtype=np.int32)), ("reversed", np.arange(M, dtype=np.int32)[::-1].copy())]
    rng = np.random.default_rng(seed)
    for i in range(n_random):
        out.append((f"shuffle{i}", rng.permutation(M).astype(np.int32)))
    return out


def build(cfg, st, perm):
    from paper_1509_05186_b200 import api
    if cfg.forest_split is not None:
        return api.Index.et_build_eforest(st["codes"], split=list(cfg.forest_split), ids=st["ids"], byte_perm=perm)
    return api.Index.et_build_etree(st["codes"], ids=st["ids"], byte_perm=perm)


def time_topk(ix, cfg, st, steps, warmup, flush):
    import torch
    q, cb = st["q_dev"], st["cb_dev"]
    for _ in range(warmup):
        d, i = ix.et_etree_topk(cfg.topk, queries=q, codebooks=cb)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        d, i = ix.et_etree_topk(cfg.topk, queries=q, codebooks=cb)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts)), d, i


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", nargs="+", default=["c2", "u1m", "c3"])
    ap.add_argument("--random", type=int, default=4)
    ap.add_argument("--seed", type=int, default=1509)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    import torch
    from paper_1509_05186_b200 import build as b, synth
    b.build()
    dev = torch.device("cuda", 0)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    rows = []
    for name in a.configs:
        cfg = synth.CONFIGS[name]
        assert not cfg.ivf_nlist and cfg.topk, "ordering study: flat top-k configs only"
        st = bench.prepare(cfg, {}, bench.CudaBackend(dev), bench.Comm(0, 1), "none")
        st["q_dev"] = torch.from_numpy(st["qx"]).to(dev)
        st["cb_dev"] = torch.from_numpy(st["cb"]).to(dev)
        ref = None
        for oname, perm in orders(cfg.M, a.random, a.seed):
            ix = build(cfg, st, perm)
            sts = ix.stats()
            ms, d, i = time_topk(ix, cfg, st, a.steps, a.warmup, flush)
            d = d.cpu().numpy()
            if ref is None:
                ref = d
            rel = float(np.max(np.abs(d - ref) / np.maximum(np.abs(ref), 1e-30)))
            L1 = sum(s["L1"] for s in sts)
            L2 = sum(s["L2"] for s in sts)
            post = sum(s["total_postfix"] for s in sts)
            look = sum(s["lookups"] for s in sts)
            rows.append((name, oname, " ".join(map(str, perm.tolist())), L1, L2, post / max(L2, 1),
                         look / (cfg.N * cfg.M), ms, rel))
            print(rows[-1], flush=True)
            ix.free()
    lines = ["| config | order | chunk permutation | L1 (internal) | L2 (leaves) | avg postfix | "
             "lookups / (N·M) | top-k step (ms) | max rel diff of top-k dist vs original |",
             "|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r[0]} | {r[1]} | {r[2]} | {r[3]} | {r[4]} | {r[5]:.3f} | {r[6]:.4f} | {r[7]:.4f} | {r[8]:.1e} |")
    txt = "\n".join(lines)
    print(txt)
    if a.out:
        with open(a.out, "w") as f:
            f.write(txt + "\n")


if __name__ == "__main__":
    main()
