#!/usr/bin/env python
"""Benchmark of the E-Tree / E-Forest ADC hot path (arXiv 1509.05186) on B200.

One step = one pass of the whole hot path over one batch of queries:
distance tables (fused into the scan kernel) -> leaf-major Distance-Context
scan -> fused top-k -> finalize (and, for N>1, the NCCL all-gather of the
per-shard lists + merge).  Default workload: BASELINE configs[1] ("c2": N=1e6
8-byte codes, Q=1e4, top-100).  Prints ONE JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1509_05186_b200 import synth  # noqa: E402

METRIC = "query·code ADC distances/sec via E-Tree/E-Forest (1M×8B codes); % of roofline"
UNIT = "distances/s"
L2_FLUSH_BYTES = 512 << 20


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured (MEASURED_PEAKS.json)"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock + throttle reasons via NVML in a background thread."""

    def __init__(self, index=0, period=0.0005):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self.period = period
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover
            log("nvml unavailable:", e)
            self.N = None

    _NAMES = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM))
                r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self._NAMES.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.N is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------- workload

def workload_config(name):
    cfg = synth.CONFIGS[name]
    return cfg


def _gen_chunk(args):
    """Worker: base vectors [s, s + n) of config ``name`` (block-addressed, so
    any worker can produce any range)."""
    name, s, n = args
    cfg = synth.CONFIGS[name]
    return s, synth.base(cfg, s, n, means=_gen_chunk.means)


def _gen_init(name):
    _gen_chunk.means = synth.mixture_means(synth.CONFIGS[name])


def gen_base_encode(cfg, cb_dev, means, dev, chunk=1 << 18):
    """Generate the base on the host block by block (a process pool for large
    N: 10^8 x 128 is ~11 min on one core), encode each block on the GPU with
    et_encode; returns host uint8 codes [N, M]."""
    import torch
    from paper_1509_05186_b200 import api
    codes = np.empty((cfg.N, cfg.M), dtype=np.uint8)
    jobs = [(cfg.name, s, min(chunk, cfg.N - s)) for s in range(0, cfg.N, chunk)]
    workers = min(len(jobs), max(1, (os.cpu_count() or 1) - 1), 48)
    if cfg.N >= (1 << 23) and workers > 1 and synth.CONFIGS.get(cfg.name) == cfg:
        import multiprocessing as mp
        with mp.get_context("spawn").Pool(workers, initializer=_gen_init, initargs=(cfg.name,)) as pool:
            for s, x in pool.imap(_gen_chunk, jobs, chunksize=1):
                xd = torch.from_numpy(x).to(dev)
                codes[s:s + len(x)] = api.et_encode(cb_dev, xd).cpu().numpy()
        return codes
    for _, s, n in jobs:
        x = torch.from_numpy(synth.base(cfg, s, n, means=means)).to(dev)
        codes[s:s + n] = api.et_encode(cb_dev, x).cpu().numpy()
    return codes


def prepare_ivf(cfg, dev, rank, world, chunk=1 << 18):
    """c4: coarse k-means (K'), residual PQ, per-list E-Trees (product path only)."""
    import torch
    from paper_1509_05186_b200 import api
    t0 = time.time()
    means = synth.mixture_means(cfg)
    coarse, _ = api.et_build_coarse(synth.coarse_train(cfg, means=means), cfg.ivf_nlist, cfg.lloyd_iters,
                                    seed=synth.kmeanspp_seed(cfg, 1))
    cdev = torch.from_numpy(coarse).to(dev)
    rt = torch.from_numpy(synth.resid_train(cfg, means=means)).to(dev)
    a = api.et_assign(cdev, rt).long()
    R = (rt - cdev[a]).cpu().numpy()
    cb, _ = api.et_build_codebooks(R, cfg.M, cfg.K, cfg.lloyd_iters, seed=synth.kmeanspp_seed(cfg, 2))
    cb_dev = torch.from_numpy(cb).to(dev)
    codes = np.empty((cfg.N, cfg.M), dtype=np.uint8)
    list_of = np.empty(cfg.N, dtype=np.int32)
    for s in range(0, cfg.N, chunk):
        n = min(chunk, cfg.N - s)
        x = torch.from_numpy(synth.base(cfg, s, n, means=means)).to(dev)
        asg = api.et_assign(cdev, x)
        codes[s:s + n] = api.et_encode(cb_dev, x, centroids=cdev, assign=asg).cpu().numpy()
        list_of[s:s + n] = asg.cpu().numpy()
    slots = np.arange(cfg.N, dtype=np.int32)
    if world > 1:   # shard whole inverted lists (LPT on list size)
        sizes = np.bincount(list_of, minlength=cfg.ivf_nlist)
        owner = np.zeros(cfg.ivf_nlist, dtype=np.int64)
        load = np.zeros(world)
        for c in np.argsort(-sizes, kind="stable"):
            r = int(np.argmin(load))
            owner[c] = r
            load[r] += sizes[c]
        m = owner[list_of] == rank
        codes, slots, list_of = codes[m], slots[m], list_of[m]
    ix = api.Index.et_build_ivf(codes, list_of, coarse, cb, ids=slots)
    qx = synth.queries(cfg, means=means)
    log(f"[rank {rank}] IVF prepared in {time.time() - t0:.1f}s: N_local={len(codes)} stats={ix.stats()}")
    sizes = np.bincount(list_of, minlength=cfg.ivf_nlist)
    return dict(cb=cb, cb_dev=cb_dev, codes=codes, ix=ix, qx=qx, coarse=coarse, list_sizes=sizes,
                q_dev=torch.from_numpy(qx).to(dev))


def prepare_ours(cfg, dev, rank, world):
    import torch
    from paper_1509_05186_b200 import api
    if cfg.ivf_nlist:
        return prepare_ivf(cfg, dev, rank, world)
    t0 = time.time()
    means = synth.mixture_means(cfg)
    cb, hist = api.et_build_codebooks(synth.train(cfg, means=means), cfg.M, cfg.K, cfg.lloyd_iters,
                                      seed=synth.kmeanspp_seed(cfg))
    cb_dev = torch.from_numpy(cb).to(dev)
    if cfg.uniform_codes:
        codes = synth.uniform_codes(cfg)
    else:
        codes = gen_base_encode(cfg, cb_dev, means, dev)
    slots = np.arange(cfg.N, dtype=np.int32)
    if world > 1:   # shard by first-level subtree (first code byte), SURVEY §8e
        hist0 = np.bincount(codes[:, 0], minlength=256)
        below = np.concatenate(([0], np.cumsum(hist0)))
        b = [0]
        for r in range(1, world):
            v = int(np.searchsorted(below, r * cfg.N / world, side="left"))
            b.append(max(b[-1], min(v, 256)))
        b.append(256)
        m = (codes[:, 0] >= b[rank]) & (codes[:, 0] < b[rank + 1])
        codes, slots = codes[m], slots[m]
    if cfg.forest_split is not None:
        ix = api.Index.et_build_eforest(codes, split=list(cfg.forest_split), ids=slots)
    else:
        ix = api.Index.et_build_etree(codes, ids=slots)
    qx = synth.queries(cfg, means=means)
    log(f"[rank {rank}] prepared in {time.time() - t0:.1f}s: N_local={len(codes)} stats={ix.stats()}")
    return dict(cb=cb, cb_dev=cb_dev, codes=codes, ix=ix, qx=qx,
                q_dev=torch.from_numpy(qx).to(dev))


def roofline(cfg, stats, kern_ms, peaks, clock_mhz, Q, n_tables=None, lookups=None):
    """Roofline of the dominant kernel (the fused table-build + scan kernel).

    Two resources bound it: the fp32 ALU of the direct-difference
    table build -- 2 lane ops (FADD + FFMA) per (table, codeword, dimension),
    peak 148 SMs x 128 lanes x max clock -- and the shared-memory lookups of the
    scan -- L1+L2+postfix per table, peak 148 SMs x 32 conflict-free 4-byte
    lookups per clock.  The larger algorithmic time is the bound reported."""
    n_tables = Q if n_tables is None else n_tables
    clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    ops = 2.0 * n_tables * cfg.K * cfg.d
    alu_peak = 148 * 128 * clk
    lk = lookups if lookups is not None else sum(s["lookups"] for s in stats) * Q
    smem_peak = 148 * 32 * clk
    sec = kern_ms / 1e3
    if ops / alu_peak >= lk / smem_peak:
        achieved, peak = ops / sec / 1e12, alu_peak / 1e12
        out = {"bound": "alu", "unit": "TFLOP/s",
               "note": "flop = one fp32 lane op (FADD or FFMA) of the table build; 2*tables*K*d per launch; "
                       "peak = 148 SM x 128 lanes x sm_max_mhz"}
    else:
        achieved, peak = lk / sec / 1e12, smem_peak / 1e12
        out = {"bound": "smem", "unit": "Tlookup/s",
               "note": "lookups = (L1+L2+postfix) per table; peak = 148 SM x 32 lookups/clk x sm_max_mhz"}
    out.update({"achieved": round(achieved, 4), "peak": round(peak, 4), "frac": round(achieved / peak, 4),
                "traffic": None, "kernel": "scan_kernel (fused tables + Distance-Context scan + top-k candidates)",
                "alu_ops": ops, "lookups": lk})
    return out


def north_star_roofline(cfg, stats, step_ms, peaks, Q, n_tables=None, lookups=None):
    """BASELINE north_star's narrow roofline: max(tree bytes / HBM, lookups /
    shared-memory rate) and the complete one (+ tables built + output).
    IVF: n_tables = Q * nprobe residual tables, lookups over the probed lists
    only (passed in); full output (topk == 0): the Q x N fp32 matrix."""
    hbm = float(peaks.get("hbm_gbs", 6558.1)) * 1e9
    clk = float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    smem_rate = 148 * 32 * clk                       # conflict-free 4-byte lookups / s
    alu = 148 * 128 * clk
    n_tables = Q if n_tables is None else n_tables
    if lookups is None:
        lookups = sum(s["lookups"] for s in stats) * Q
        if len(stats) > 1:
            lookups += stats[0]["groups"] * Q         # one join add per tuple
    tree_bytes = sum(s["device_bytes"] for s in stats)
    t_tree = tree_bytes / hbm
    t_smem = lookups / smem_rate
    t_lut_build = 2.0 * n_tables * cfg.K * cfg.d / alu
    t_out = (Q * cfg.N * 4 if cfg.topk == 0 else Q * cfg.topk * 8) / hbm
    narrow = max(t_tree, t_smem)
    complete = max(t_tree + t_out, t_smem, t_lut_build)
    s = step_ms / 1e3
    return {"narrow_us": round(narrow * 1e6, 3), "complete_us": round(complete * 1e6, 3),
            "frac_narrow": round(narrow / s, 4), "frac_complete": round(complete / s, 4),
            "terms_us": {"tree_bytes": round(t_tree * 1e6, 3), "smem_lookups": round(t_smem * 1e6, 3),
                         "table_build_alu": round(t_lut_build * 1e6, 3), "topk_out": round(t_out * 1e6, 3)},
            "lookups_per_query": int(lookups // Q), "tree_bytes": tree_bytes}


def cpu_baseline(cfg, cb, codes, qx, budget_s=15.0):
    """The oracle as it stands (naive ADC in fp64 + exact top-k by full sort) on
    a bounded sample of the workload's queries, host cores."""
    from oracle import pq, topk
    n = 0
    t0 = time.perf_counter()
    ids = np.arange(len(codes))
    while True:
        table = pq.lut64(cb, qx[n:n + 1])
        dist = pq.adc(table, codes)
        topk.topk(dist, ids, cfg.topk)
        n += 1
        el = time.perf_counter() - t0
        if el >= budget_s or n >= len(qx):
            break
    return {"value": n * len(codes) / el, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{n} queries x {len(codes)} codes (oracle naive ADC fp64 + full-sort top-{cfg.topk}), "
                      f"{el:.1f}s"}


# --------------------------------------------------------------------------- our arm

def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_1509_05186_b200 import api, build as _build
    rank, world, local = dist_env()
    _build.build()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = workload_config(args.config)
    Q, k = cfg.Q, cfg.topk
    st = prepare_ours(cfg, dev, rank, world)
    ix, qd, cbd = st["ix"], st["q_dev"], st["cb_dev"]
    stats = ix.stats()
    kk = max(k, 1)
    dist_out = torch.empty((Q, kk), dtype=torch.float32, device=dev)
    ids_out = torch.empty((Q, kk), dtype=torch.int32, device=dev)
    if world > 1:
        gd = torch.empty((world, Q, kk), dtype=torch.float32, device=dev)
        gi = torch.empty((world, Q, kk), dtype=torch.int32, device=dev)

    full = (k == 0)
    ivf = bool(cfg.ivf_nlist)
    if full:
        full_out = torch.empty((Q, ix.N), dtype=torch.float32, device=dev)

    def local_step(q_in):
        if full:
            return ix.et_etree_distances(queries=q_in, codebooks=cbd, out=full_out)
        if ivf:
            d_, i_ = ix.et_ivf_topk(q_in, nprobe=cfg.ivf_nprobe, k=k)
            dist_out.copy_(d_)
            ids_out.copy_(i_)
            return dist_out, ids_out
        return ix.et_etree_topk(k, queries=q_in, codebooks=cbd, out=(dist_out, ids_out))

    def step():
        r = local_step(qd)
        if world > 1 and not full:
            dist.all_gather_into_tensor(gd, dist_out)
            dist.all_gather_into_tensor(gi, ids_out)
            return api.et_merge_topk(gd, gi)
        return r

    # query.code pairs per step (IVF: sum of the probed lists' sizes)
    if ivf:
        _, _, pr = ix.et_ivf_topk(qd, nprobe=cfg.ivf_nprobe, k=k, return_probes=True)
        pairs = int(st["list_sizes"][pr.cpu().numpy().ravel()].sum())
        if world > 1:
            t = torch.tensor([pairs], device=dev, dtype=torch.float64)
            dist.all_reduce(t)
            pairs = int(t.item())
    else:
        pairs = Q * cfg.N
    k_alloc = max(k, 1)

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device=dev)
    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    l0 = api.et_launch_count()
    step()
    torch.cuda.synchronize()
    launches_per_step = api.et_launch_count() - l0

    graph = None
    if world == 1:
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            step()
        torch.cuda.current_stream().wait_stream(s)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step()
        for _ in range(3):
            graph.replay()
    run = graph.replay if graph is not None else step

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for a, b in evs:
            flush.fill_(1.0)            # untimed: evict L2 between timed steps
            a.record()
            run()
            b.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    step_ms = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    if world > 1:
        t = torch.tensor([step_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_ms = float(t.item())
    value = pairs / (step_ms / 1e3)

    # per-kernel breakdown: the same steps, library events around each launch
    api.et_timing_reset()
    api.et_timing_enable(True)
    for _ in range(args.steps):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    kern = {}
    for name in ("fill", "probe", "bucket", "scan", "finalize", "luts", "gather"):
        ms, n = api.et_timing_get(name)
        if n:
            kern[name] = ms / n
    api.et_timing_enable(False)
    dom = max(kern, key=kern.get)

    # e2e: host (pinned) queries in, top-k out, copies inside the timed region
    qh = torch.from_numpy(st["qx"]).pin_memory()
    out_shape = (Q, cfg.N) if full else (Q, kk)
    dh = torch.empty(out_shape, dtype=torch.float32).pin_memory()
    ih = torch.empty((Q, kk), dtype=torch.int32).pin_memory()
    q_stage = torch.empty_like(qd)
    e_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
             for _ in range(max(5, args.steps // 4))]
    torch.cuda.synchronize()
    for a, b in e_evs:
        flush.fill_(1.0)
        a.record()
        q_stage.copy_(qh, non_blocking=True)
        r = local_step(q_stage)
        if full:
            dh.copy_(r, non_blocking=True)
        else:
            if world > 1:
                dist.all_gather_into_tensor(gd, dist_out)
                dist.all_gather_into_tensor(gi, ids_out)
                md, mi = api.et_merge_topk(gd, gi)
            else:
                md, mi = dist_out, ids_out
            dh.copy_(md, non_blocking=True)
            ih.copy_(mi, non_blocking=True)
        b.record()
    torch.cuda.synchronize()
    e2e_ms = sum(a.elapsed_time(b) for a, b in e_evs) / len(e_evs)
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    peaks, peak_src = load_peaks()
    if rank == 0:
        if full and kern.get("gather", 0) > kern.get("scan", 0):
            hbm = float(peaks.get("hbm_gbs", 6558.1))
            byts = Q * cfg.N * 4 + cfg.N * 4
            ach = byts / (kern["gather"] / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(ach / hbm, 4), "traffic": None,
                    "kernel": "gather_full_kernel (Q x N fp32 output write)",
                    "note": "algorithmic bytes = 4*Q*N output + 4*N slot->leaf map"}
            dom_ms = kern["gather"]
        else:
            n_tables = Q * cfg.ivf_nprobe if ivf else Q
            lookups = None
            if ivf:
                lookups = stats[0]["lookups"] / max(1, cfg.N) * pairs
            roof = roofline(cfg, stats, kern["scan"], peaks, clk.summary()["sm_mhz"], Q, n_tables, lookups)
            dom_ms = kern["scan"]
        roof["peak_source"] = peak_src
        roof["share_of_step"] = round(dom_ms / sum(kern.values()), 4)
        tr = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tr):
            with open(tr) as f:
                t = json.load(f).get(args.config, {}).get("scan")
            roof["traffic"] = t
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": (f"{cfg.name}: BASELINE configs[{['c1','c2','c3','c4','c5'].index(cfg.name)}]"
                                    if cfg.name in ['c1', 'c2', 'c3', 'c4', 'c5'] else f"{cfg.name}: diagnostic companion"),
                       "pairs_per_step": pairs,
                       "N": cfg.N, "d": cfg.d, "M": cfg.M, "K": cfg.K, "Q": Q, "k": k,
                       "forest_split": cfg.forest_split,
                       "parallelism": f"db-shard{world} (first-level subtrees) + all-gather" if world > 1 else "1 GPU",
                       "l2": f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write)",
                       "timing": "CUDA graph replay of one step, CUDA events per step" if world == 1 else "CUDA events per step"},
            "roofline": roof,
            "north_star_roofline": north_star_roofline(cfg, stats, step_ms, peaks, Q,
                                                       Q * cfg.ivf_nprobe if ivf else None,
                                                       stats[0]["lookups"] / max(1, cfg.N) * pairs if ivf else None),
            "kernels_ms": {k_: round(v, 5) for k_, v in kern.items()},
            "dominant_kernel": dom,
            "e2e": {"value": pairs / (e2e_ms / 1e3), "unit": UNIT,
                    "h2d_bytes_per_step": int(qh.numel() * 4),
                    "d2h_bytes_per_step": int(dh.numel() * 4 + (0 if full else ih.numel() * 4)),
                    "ms_per_step": e2e_ms},
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clk.summary(),
            "tree_stats": [{kk: s[kk] for kk in ("L1", "L2", "total_postfix", "lookups", "paper_bytes")} for s in stats],
        }
        if world == 1 and not args.no_cpu_baseline and not ivf:
            out["cpu_baseline"] = cpu_baseline(cfg, st["cb"], st["codes"], st["qx"])
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------------------- reference arm

def run_reference(args):
    """The oracle (plain numpy) timed on the host cores on the same workload:
    each step is a bounded sample (one query against all N codes)."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from oracle import pq, topk
    cfg = workload_config(args.config)
    t0 = time.time()
    means = synth.mixture_means(cfg)
    cb, _ = pq.train_pq(synth.train(cfg, means=means), cfg.M, cfg.K, cfg.lloyd_iters, synth.kmeanspp_seed(cfg))
    if cfg.uniform_codes:
        codes = synth.uniform_codes(cfg)
    else:
        codes = np.concatenate([pq.encode(cb, synth.base(cfg, s, min(1 << 18, cfg.N - s), means=means))
                                for s in range(0, cfg.N, 1 << 18)])
    qx = synth.queries(cfg, means=means)
    log(f"[reference] oracle inputs prepared in {time.time() - t0:.1f}s")
    ids = np.arange(cfg.N)
    per_step_q = 1

    def step(i):
        q = (i * per_step_q) % cfg.Q
        table = pq.lut64(cb, qx[q:q + per_step_q])
        topk.topk(pq.adc(table, codes), ids, cfg.topk)

    for i in range(args.warmup):
        step(i)
    t = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    el = time.perf_counter() - t
    ms = el / args.steps * 1e3
    value = per_step_q * cfg.N / (ms / 1e3)
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": f"{cfg.name}", "N": cfg.N, "d": cfg.d, "M": cfg.M, "K": cfg.K,
                      "Q_per_step": per_step_q, "k": cfg.topk},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"{per_step_q} query x {cfg.N} codes per step (naive ADC fp64 + full-sort top-k)"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
