"""Run a few hot-path steps of one config (for ncu / compute-sanitizer captures).

  python tools/prof_step.py --config c2 --steps 5
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--Q", type=int, default=0)
    a = ap.parse_args()
    import torch
    from paper_1509_05186_b200 import build, synth
    build.build()
    cfg = synth.CONFIGS[a.config]
    if a.Q:
        cfg = synth.scaled(cfg, Q=a.Q)
    dev = torch.device("cuda", 0)
    st = bench.prepare(cfg, {}, bench.CudaBackend(dev), bench.Comm(0, 1), "none")
    ix = bench.build_index(cfg, st)
    st["q_dev"] = torch.from_numpy(st["qx"]).to(dev)
    st["cb_dev"] = torch.from_numpy(st["cb"]).to(dev)
    for _ in range(a.steps):
        if cfg.ivf_nlist:
            d, i = ix.et_ivf_topk(st["q_dev"], nprobe=cfg.ivf_nprobe, k=cfg.topk)
        elif cfg.topk == 0:   # full Q x N output (c1)
            d = ix.et_etree_distances(queries=st["q_dev"], codebooks=st["cb_dev"])
            i = d[:, :4].int()
        else:
            d, i = ix.et_etree_topk(cfg.topk, queries=st["q_dev"], codebooks=st["cb_dev"])
    torch.cuda.synchronize()
    print("ok", d[0, :4].tolist(), i[0, :4].tolist())


if __name__ == "__main__":
    main()
