"""Small invocations of every hot-path shape, for compute-sanitizer runs.

  compute-sanitizer --tool memcheck   python tools/sanitize_cases.py
  compute-sanitizer --tool racecheck  python tools/sanitize_cases.py
  compute-sanitizer --tool synccheck  python tools/sanitize_cases.py

Cases (scaled so the sanitizers finish in minutes): c1 full output and top-k
(8-level tree, TMEM levels), U1M-like uniform codes with S > 1 segments
(qthr seeding, candidate refresh + compaction), a c3-shape joined forest
(M = 16, s = 60), a c5-shape fused forest (M = 8, split 0-3 | 4-7), a 4-level
tree (all levels in shared memory), IVF (probe, two-tier bucketing, residual
tables) and the shard merge.  Each result is checked against the oracle
(test infrastructure) so a sanitizer-clean run is also a correct one.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    import torch
    from oracle import ivf as oivf
    from oracle import pq
    from paper_1509_05186_b200 import api, build, synth
    from gpu_common import check_topk

    build.build()
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731

    def small(seed, N, M, K, s, Q, nd=None):
        codes = synth.random_codes(seed, N, M, K, nd)
        cb = synth.random_floats(seed + 1, (M, K, s), 0, 10)
        qx = synth.random_floats(seed + 2, (Q, M * s), 0, 10)
        return cb, codes, qx

    # c1-like: 8-level tree, full output + top-k
    cb, codes, qx = small(1, 20_000, 8, 256, 16, 40, nd=600)
    ix = api.Index.et_build_etree(codes)
    full = ix.et_etree_distances(queries=dev(qx), codebooks=dev(cb))
    d, i = ix.et_etree_topk(50, queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    ref = pq.adc(pq.lut64(cb, qx), codes)
    assert (np.abs(full.cpu().numpy() - ref) / np.maximum(ref, 1e-30)).max() <= 1e-5
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, 50, range(len(qx)))
    print("c1-like ok")

    # U1M-like: uniform codes, several segments per chunk
    codes = synth.uniform_codes(synth.CONFIGS["u1m"], 120_000)
    cb2 = synth.random_floats(5, (8, 256, 16), 0, 10)
    qx2 = synth.random_floats(6, (48, 128), 0, 10)
    ix = api.Index.et_build_etree(codes)
    d, i = ix.et_etree_topk(100, queries=dev(qx2), codebooks=dev(cb2))
    torch.cuda.synchronize()
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb2, qx2, codes, 100, range(0, 48, 5))
    print("u1m-like ok")

    # c3-shape joined forest (M = 16, s = 60)
    cb, codes, qx = small(11, 8_000, 16, 256, 60, 12, nd=400)
    ix = api.Index.et_build_eforest(codes, split=[0, 8, 16])
    d, i = ix.et_etree_topk(20, queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, 20, range(len(qx)))
    print("c3-like ok")

    # c5-shape fused forest (M = 8, split 0-3 | 4-7) and a 3-tree split
    cb, codes, qx = small(21, 30_000, 8, 256, 16, 40, nd=3000)
    for split in ([0, 4, 8], [0, 3, 5, 8]):
        ix = api.Index.et_build_eforest(codes, split=split)
        d, i = ix.et_etree_topk(100, queries=dev(qx), codebooks=dev(cb))
        torch.cuda.synchronize()
        check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, 100, range(0, 40, 3))
    print("c5-like ok")

    # 4-level tree (every level in shared memory), K < 256
    cb, codes, qx = small(31, 5_000, 4, 16, 4, 33)
    ix = api.Index.et_build_etree(codes, K=16)
    d, i = ix.et_etree_topk(10, queries=dev(qx), codebooks=dev(cb))
    torch.cuda.synchronize()
    check_topk(d.cpu().numpy(), i.cpu().numpy(), cb, qx, codes, 10, range(len(qx)))
    print("4-level ok")

    # IVF (c4 shape, scaled)
    cfg = synth.scaled(synth.CONFIGS["c4"], N=30_000, Q=24, n_train=4_000, n_coarse_train=4_000,
                       ivf_nlist=16, lloyd_iters=3)
    means = synth.mixture_means(cfg)
    coarse, _ = pq.kmeans(synth.coarse_train(cfg, means=means), 16, 3, 7)
    rt = synth.resid_train(cfg, means=means)
    a = pq.assign(rt, coarse)
    cbr, _ = pq.train_pq((rt - coarse[a]).astype(np.float32), 8, 256, 3, 8)
    index = oivf.encode_ivf(synth.base(cfg, means=means), coarse.astype(np.float32), cbr)
    qx = synth.queries(cfg, means=means)
    ix = api.Index.et_build_ivf(index.codes, index.assign.astype(np.int32), index.coarse, index.codebooks)
    d, i, pr = ix.et_ivf_topk(dev(qx), nprobe=4, k=20, return_probes=True)
    torch.cuda.synchronize()
    D, I, _ = oivf.search(index, qx, 4, 20, probes=pr.cpu().numpy())
    dd = d.cpu().numpy()
    assert np.all(np.abs(dd - D) <= 1e-5 * np.maximum(D, 1e-30))
    print("ivf ok")

    # shard merge (K7)
    gd = torch.rand(3, 16, 20, device="cuda").sort(dim=2).values
    gi = torch.randint(0, 1000, (3, 16, 20), device="cuda", dtype=torch.int32)
    md, mi = api.et_merge_topk(gd, gi)
    torch.cuda.synchronize()
    print("merge ok")
    print("ALL OK")


if __name__ == "__main__":
    main()
