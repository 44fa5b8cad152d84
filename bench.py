#!/usr/bin/env python
"""Benchmark of the E-Tree / E-Forest ADC hot path (arXiv 1509.05186) on B200.

One step = one pass of the whole hot path over one batch of queries:
distance tables (fused into the scan kernel) -> leaf-major Distance-Context
scan -> fused top-k -> finalize, and for a database sharded over N > 1 GPUs
the NCCL all-gather of the per-shard lists + merge.  Default workload:
BASELINE configs[1] ("c2": N=1e6 8-byte codes, Q=1e4, top-100).  Prints ONE
JSON line (rank 0).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c1..c5|u1m]
                  [--impl ours|reference] [--shard auto|db|queries|lists]

Multi-GPU.  ``--gpus N`` without a torchrun
environment re-launches this script under ``torch.distributed.run`` with N
ranks (one per GPU); under torchrun, WORLD_SIZE must equal N.  Shard modes:
  db      -- the database split by first-level subtree (first code byte, the
             cut of et_shard_bounds), queries broadcast, per-shard
             top-k all-gathered (NCCL) and merged (et_merge_topk).  Each rank
             generates and encodes 1/N of the base and the codes are exchanged
             by first byte (all-to-all), so no rank touches the whole base.
  lists   -- IVF (c4): whole inverted lists per rank (et_shard_lists, LPT),
             same gather + merge.
  queries -- the index replicated, the queries split; no collective on the
             data path (a tiny database: c1/c2/u1m).
``auto`` = db for the forest configs (c3, c5; BASELINE names them sharded),
lists for c4, queries otherwise.

The oracle legs (``cpu_baseline``, the ``parity`` check and ``--impl
reference``) are the only places this script runs ``oracle/`` code.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import statistics
import subprocess
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
CFG_INDEX = {"c1": 0, "c2": 1, "c3": 2, "c4": 3, "c5": 4}


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


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def relaunch_if_needed(args):
    """--gpus N > 1 outside torchrun: re-exec under torch.distributed.run (one
    rank per GPU).  Under torchrun: the world size must equal --gpus."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1:
        return
    if not args.dry_run:
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but only {n} CUDA device(s) visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    log("[bench] launching:", " ".join(cmd))
    raise SystemExit(subprocess.call(cmd))


# --------------------------------------------------------------------------- clocks

class ClockSampler:
    """Samples SM clock + throttle reasons via NVML in a background thread."""

    _NAMES = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index=0, period=0.0005):
        self.samples, self.reasons, self.max_mhz, self.period = [], set(), None, period
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


# --------------------------------------------------------------------------- communication helpers

class Comm:
    """Thin wrapper of torch.distributed for the host-side plumbing (NCCL on
    the GPU box, gloo in the CPU dry run); world 1 = no-ops."""

    def __init__(self, rank, world, device=None):
        self.rank, self.world, self.device = rank, world, device
        self.nccl = False
        if world > 1:
            import torch.distributed as dist
            self.dist = dist
            self.nccl = dist.get_backend() == "nccl"

    def _t(self, arr):
        import torch
        t = torch.from_numpy(np.ascontiguousarray(arr))
        return t.to(self.device) if self.nccl else t

    def bcast(self, arr, src=0):
        if self.world == 1:
            return arr
        t = self._t(arr)
        self.dist.broadcast(t, src)
        return t.cpu().numpy()

    def allsum(self, arr):
        if self.world == 1:
            return arr
        t = self._t(arr)
        self.dist.all_reduce(t)
        return t.cpu().numpy()

    def allmax(self, x: float) -> float:
        if self.world == 1:
            return x
        t = self._t(np.array([x], np.float64))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.cpu().numpy()[0])

    def allgather(self, arr):
        """Same-shape arrays from every rank -> [world, ...]."""
        import torch
        if self.world == 1:
            return np.asarray(arr)[None]
        t = self._t(arr)
        if self.nccl:
            out = torch.empty((self.world, *t.shape), dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, t)
            return out.cpu().numpy()
        lst = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(lst, t)
        return torch.stack(lst).numpy()

    def exchange(self, parts):
        """All-to-all of host arrays: parts[r] goes to rank r; returns the
        concatenation of what every rank sent here (rank order)."""
        import torch
        if self.world == 1:
            return parts[0]
        counts = np.array([len(p) for p in parts], np.int64)
        cm = self.allgather(counts)                      # cm[src][dst]
        recv = cm[:, self.rank]
        tail = parts[0].shape[1:]
        dtype = parts[0].dtype
        send = np.concatenate(parts) if sum(counts) else np.zeros((0, *tail), dtype)
        if self.nccl:
            st = self._t(send.reshape(len(send), -1) if send.ndim > 1 else send)
            out = torch.empty((int(recv.sum()), *st.shape[1:]), dtype=st.dtype, device=st.device)
            self.dist.all_to_all_single(out, st, output_split_sizes=recv.tolist(), input_split_sizes=counts.tolist())
            return out.cpu().numpy().reshape((-1, *tail))
        # gloo has no all-to-all: pairwise send/recv rounds
        offs = np.concatenate(([0], np.cumsum(counts)))
        got = [None] * self.world
        got[self.rank] = parts[self.rank]
        for step in range(1, self.world):
            to, fr = (self.rank + step) % self.world, (self.rank - step) % self.world
            buf = torch.empty((int(recv[fr]), *tail), dtype=torch.from_numpy(send[:0]).dtype)
            reqs = []
            if counts[to]:
                reqs.append(self.dist.isend(torch.from_numpy(np.ascontiguousarray(send[offs[to]:offs[to + 1]])), to))
            if recv[fr]:
                reqs.append(self.dist.irecv(buf, fr))
            for r_ in reqs:
                r_.wait()
            got[fr] = buf.numpy()
        return np.concatenate(got)


# --------------------------------------------------------------------------- backends

class CudaBackend:
    """The product path: every compute step runs in libetree.so's kernels."""
    name = "cuda"

    def __init__(self, dev):
        from paper_1509_05186_b200 import api
        self.api, self.dev = api, dev

    def _d(self, a):
        import torch
        return torch.from_numpy(np.ascontiguousarray(a)).to(self.dev)

    def train_codebooks(self, X, M, K, iters, seed):
        return self.api.et_build_codebooks(X, M, K, iters, seed=seed)[0]

    def train_coarse(self, X, nlist, iters, seed):
        return self.api.et_build_coarse(X, nlist, iters, seed=seed)[0]

    def encode(self, cb, X, coarse=None):
        """codes (and the coarse cell, IVF) of host vectors X."""
        cbd, xd = self._d(cb), self._d(X)
        if coarse is None:
            return self.api.et_encode(cbd, xd).cpu().numpy(), None
        cd = self._d(coarse)
        a = self.api.et_assign(cd, xd)
        return self.api.et_encode(cbd, xd, centroids=cd, assign=a).cpu().numpy(), a.cpu().numpy()

    def assign(self, coarse, X):
        return self.api.et_assign(self._d(coarse), self._d(X)).long().cpu().numpy()


def _gen_chunk(args):
    """Worker: base vectors [s, s + n) of config ``name`` (block-addressed)."""
    name, over, s, n = args
    cfg = synth.scaled(synth.CONFIGS[name], **over) if over else synth.CONFIGS[name]
    return s, synth.base(cfg, s, n, means=_gen_chunk.means)


def _gen_init(name, over):
    cfg = synth.scaled(synth.CONFIGS[name], **over) if over else synth.CONFIGS[name]
    _gen_chunk.means = synth.mixture_means(cfg)


def gen_encode_range(cfg, over, backend, cb, means, lo, hi, coarse=None, chunk=1 << 18, workers=None):
    """Generate base vectors [lo, hi) block by block (a process pool for large
    ranges) and encode each block with ``backend``; returns (codes, cells)."""
    n = hi - lo
    codes = np.empty((n, cfg.M), dtype=np.uint8)
    cells = np.empty(n, dtype=np.int32) if coarse is not None else None
    jobs = [(cfg.name, over, s, min(chunk, hi - s)) for s in range(lo, hi, chunk)]
    if workers is None:
        workers = min(len(jobs), max(1, (os.cpu_count() or 1) - 1), 48)
    if n >= (1 << 23) and workers > 1:
        import multiprocessing as mp
        with mp.get_context("spawn").Pool(workers, initializer=_gen_init, initargs=(cfg.name, over)) as pool:
            it = pool.imap(_gen_chunk, jobs, chunksize=1)
            for s, x in it:
                c, a = backend.encode(cb, x, coarse)
                codes[s - lo:s - lo + len(x)] = c
                if cells is not None:
                    cells[s - lo:s - lo + len(x)] = a
        return codes, cells
    for _, _, s, m in jobs:
        c, a = backend.encode(cb, synth.base(cfg, s, m, means=means), coarse)
        codes[s - lo:s - lo + m] = c
        if cells is not None:
            cells[s - lo:s - lo + m] = a
    return codes, cells


def shard_mode(cfg, args, world):
    if world == 1:
        return "none"
    if args.shard != "auto":
        return args.shard
    if cfg.ivf_nlist:
        return "lists"
    return "db" if cfg.forest_split is not None else "queries"


def prepare(cfg, over, backend, comm, mode):
    """Inputs of this rank: codebooks (rank 0 trains, broadcast), its codes and
    global ids (sharded modes: each rank encodes 1/world of the base, rows are
    exchanged to their owner), queries."""
    from paper_1509_05186_b200 import api
    rank, world = comm.rank, comm.world
    t0 = time.time()
    means = synth.mixture_means(cfg)
    coarse = None
    if cfg.ivf_nlist:
        if rank == 0:
            coarse = backend.train_coarse(synth.coarse_train(cfg, means=means), cfg.ivf_nlist, cfg.lloyd_iters,
                                          synth.kmeanspp_seed(cfg, 1))
            rt = synth.resid_train(cfg, means=means)
            a = backend.assign(coarse, rt)
            cb = backend.train_codebooks((rt - coarse[a]).astype(np.float32), cfg.M, cfg.K, cfg.lloyd_iters,
                                         synth.kmeanspp_seed(cfg, 2))
        else:
            coarse = np.empty((cfg.ivf_nlist, cfg.d), np.float32)
            cb = np.empty((cfg.M, cfg.K, cfg.d // cfg.M), np.float32)
        coarse, cb = comm.bcast(coarse), comm.bcast(cb)
    else:
        cb = (backend.train_codebooks(synth.train(cfg, means=means), cfg.M, cfg.K, cfg.lloyd_iters,
                                      synth.kmeanspp_seed(cfg)) if rank == 0
              else np.empty((cfg.M, cfg.K, cfg.d // cfg.M), np.float32))
        cb = comm.bcast(cb)
    # this rank's share of the base
    if mode in ("none", "queries"):
        lo, hi = 0, cfg.N
    else:
        lo, hi = rank * cfg.N // world, (rank + 1) * cfg.N // world
    if cfg.uniform_codes:
        codes, cells = synth.uniform_codes(cfg)[lo:hi], None
    else:
        codes, cells = gen_encode_range(cfg, over, backend, cb, means, lo, hi, coarse)
    ids = np.arange(lo, hi, dtype=np.int32)
    list_sizes = None
    if cfg.ivf_nlist:
        list_sizes = comm.allsum(np.bincount(cells, minlength=cfg.ivf_nlist).astype(np.int64))
    if mode == "db":
        hist = comm.allsum(np.bincount(codes[:, 0], minlength=256).astype(np.int64))
        b = api.et_shard_bounds_hist(hist, world)
        dest = np.searchsorted(b, codes[:, 0], side="right") - 1
        parts = [np.flatnonzero(dest == r) for r in range(world)]
        codes = comm.exchange([codes[p] for p in parts])
        ids = comm.exchange([ids[p] for p in parts])
    elif mode == "lists":
        owner = api.et_shard_lists(list_sizes, world)
        dest = owner[cells]
        parts = [np.flatnonzero(dest == r) for r in range(world)]
        codes = comm.exchange([codes[p] for p in parts])
        ids = comm.exchange([ids[p] for p in parts])
        cells = comm.exchange([cells[p] for p in parts])
    qx = synth.queries(cfg, means=means)
    log(f"[rank {rank}] prepared in {time.time() - t0:.1f}s: mode={mode} N_local={len(codes)}")
    return dict(cb=cb, coarse=coarse, codes=codes, ids=ids, cells=cells, qx=qx, list_sizes=list_sizes, means=means)


def build_index(cfg, st):
    from paper_1509_05186_b200 import api
    codes, ids = st["codes"], st["ids"]
    if len(codes) == 0:
        return None
    if cfg.ivf_nlist:
        return api.Index.et_build_ivf(codes, st["cells"], st["coarse"], st["cb"], ids=ids)
    if cfg.forest_split is not None:
        return api.Index.et_build_eforest(codes, split=list(cfg.forest_split), ids=ids)
    return api.Index.et_build_etree(codes, ids=ids)


# --------------------------------------------------------------------------- rooflines

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
                "traffic": None,
                "kernel": ("narrow_kernel (fused tables of all 16 levels + masked tuple scan + top-k candidates)"
                           if cfg.forest_split and cfg.M > 8 else
                           "scan_kernel (fused tables + Distance-Context scan + top-k candidates)"),
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


# --------------------------------------------------------------------------- oracle legs

def cpu_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


_ADC_CODES = None   # set before the fork pool starts (inherited, not pickled)
_ADC_CHUNK = 1 << 22   # codes per oracle call: bounded temporaries at N = 1e8


def _adc_chunked(tables, codes):
    """The oracle's naive ADC (pq.adc) over all codes, a chunk of codes per call."""
    from oracle import pq
    for s in range(0, len(codes), _ADC_CHUNK):
        pq.adc(tables, codes[s:s + _ADC_CHUNK])


def _adc_worker(tables):
    """Pool worker (all-cores mode): naive ADC of the given queries' tables."""
    t = time.perf_counter()
    _adc_chunked(tables, _ADC_CODES)
    return time.perf_counter() - t


def cpu_baseline(cfg, st, budget_s=15.0):
    """The oracle as it stands, on the GPU box's host cores:
    (i) naive ADC (O3, fp64 tables, tables excluded from the timing) and the
    paper's HMS traversal (O6) on one thread, (ii) naive ADC with the queries
    split over every core.  ``value`` = mode (ii) in query.code pairs/s."""
    from oracle import etree, pq
    import multiprocessing as mp
    codes, qx, cb = st["codes"], st["qx"], st["cb"]
    N = len(codes)
    out = {"unit": UNIT, "kind": "oracle", **cpu_info()}
    per = max(1, budget_s / 4)
    # (a) tables alone (reported, excluded from the ADC / traversal rates)
    t = time.perf_counter()
    n = 0
    while time.perf_counter() - t < min(per, 2.0) and n < len(qx):
        pq.lut64(cb, qx[n:n + 1])
        n += 1
    out["lut64_ms_per_query"] = round((time.perf_counter() - t) / n * 1e3, 3)
    # (b) naive ADC, one thread
    tabs = pq.lut64(cb, qx[:64])
    t = time.perf_counter()
    n = 0
    while True:
        _adc_chunked(tabs[n % 64:n % 64 + 1], codes)
        n += 1
        el = time.perf_counter() - t
        if el >= per or n >= len(qx):
            break
    adc1 = n * N / el
    out["adc_1thread"] = {"value": adc1, "sample": f"{n} queries x {N} codes", "seconds": round(el, 2)}
    # (c) HMS traversal (O6), one thread, on a bounded sample of the database
    ns = min(N, 1 << 17)
    sc, sid = etree.sort_codes(codes[:ns, :min(cfg.M, 8)], np.arange(ns))
    buf = etree.serialize(etree.build_alg1(sc, sid))
    t32 = pq.lut32(cb[:min(cfg.M, 8)], qx[:64, :min(cfg.M, 8) * (cfg.d // cfg.M)])
    t = time.perf_counter()
    n = 0
    while True:
        etree.traverse(buf, min(cfg.M, 8), t32[n % 64:n % 64 + 1], ns)
        n += 1
        el = time.perf_counter() - t
        if el >= per:
            break
    out["traverse_1thread"] = {"value": n * ns / el, "sample": f"{n} queries x the first {ns} codes"
                               + (" (bytes 0-7 only)" if cfg.M > 8 else ""), "seconds": round(el, 2)}
    # (d) naive ADC, every core (queries split over a fork pool)
    global _ADC_CODES
    _ADC_CODES = codes
    cores = os.cpu_count() or 1
    qpc = 4 if N < 10_000_000 else 1          # queries per pool task
    nq = int(min(64 * cores, max(qpc * cores, per * adc1 * cores / N)))
    if N >= 10_000_000:
        nq = cores                            # one query per core (each is >= 1e7 codes)
    tabs = [pq.lut64(cb, qx[(qpc * i) % len(qx):(qpc * i) % len(qx) + qpc]) for i in range(max(1, nq // qpc))]
    t = time.perf_counter()
    with mp.get_context("fork").Pool(cores) as pool:
        pool.map(_adc_worker, tabs, chunksize=1)
    el = time.perf_counter() - t
    _ADC_CODES = None
    pairs = sum(len(tb) for tb in tabs) * N
    out["adc_all_cores"] = {"value": pairs / el, "cores": cores, "sample": f"{pairs // N} queries x {N} codes",
                            "seconds": round(el, 2)}
    out["value"] = pairs / el
    out["cores"] = cores
    out["sample"] = (f"naive ADC (fp64 tables precomputed, excluded) of {pairs // N} queries x {N} codes "
                     f"over {cores} processes")
    return out


def oracle_shard_topk(cfg, st, qsel, gpu_probes=None):
    """Exact top-k of the sampled queries over THIS rank's codes (oracle, fp64):
    full distances, then the full sort of the k-th-value superset."""
    from oracle import pq, topk
    codes, ids, k = st["codes"], st["ids"].astype(np.int64), cfg.topk
    D = np.full((len(qsel), k), np.inf)
    I = np.full((len(qsel), k), -1, np.int64)
    for j, q in enumerate(qsel):
        if len(codes) == 0:
            continue
        if cfg.ivf_nlist:
            full = np.full(len(codes), np.inf)
            for c in gpu_probes[j]:
                m = np.flatnonzero(st["cells"] == c)
                if len(m):
                    r = st["qx"][q].astype(np.float64) - st["coarse"][c].astype(np.float64)
                    full[m] = pq.adc(pq.lut64(st["cb"], r[None]), codes[m])[0]
        else:
            full = np.empty(len(codes))
            tab = pq.lut64(st["cb"], st["qx"][q:q + 1])
            for s in range(0, len(codes), 1 << 23):
                full[s:s + (1 << 23)] = pq.adc(tab, codes[s:s + (1 << 23)])[0]
        fin = np.isfinite(full)
        kk = min(k, int(fin.sum()))
        if kk == 0:
            continue
        kth = np.partition(full[fin], kk - 1)[kk - 1]
        sel = np.flatnonzero(full <= kth)
        D[j:j + 1], I[j:j + 1] = topk.topk(full[sel][None], ids[sel], k)
    return D, I


def parity_full(cfg, st, got, qsel, rtol=1e-5):
    """Full output (c1): every entry of the sampled queries' rows vs ADC64."""
    from oracle import pq
    ref = pq.adc(pq.lut64(st["cb"], st["qx"][qsel]), st["codes"])
    err = np.abs(got.astype(np.float64) - ref) / np.maximum(ref, 1e-30)
    return {"queries": len(qsel), "entries": int(ref.size), "max_rel_err": float(err.max()),
            "ok": bool(err.max() <= rtol), "protocol": "every entry of the sampled rows within 1e-5 rel of fp64 ADC"}


def parity_check(cfg, st, comm, gd, gi, qsel, gpu_probes=None, rtol=1e-5):
    """GPU top-k of the sampled queries vs the oracle's (C1/C2 of DESIGN.md
    §3.C).  Each rank computes the oracle's exact top-k over its own shard;
    the lists are merged on rank 0 (the oracle's shard simulation O10)."""
    from oracle import topk
    probe_swaps = 0
    if gpu_probes is not None:   # C6: the GPU's probes may differ from the oracle's only at near ties
        from oracle import ivf as oivf, pq
        op = oivf.probe(st["qx"][qsel], st["coarse"], cfg.ivf_nprobe)
        cd = pq.sqdist_direct(st["qx"][qsel], st["coarse"])
        for j in range(len(qsel)):
            diff = set(gpu_probes[j].tolist()) ^ set(op[j].tolist())
            kth = np.sort(cd[j])[cfg.ivf_nprobe - 1]
            probe_swaps += len(diff)
            if any(abs(cd[j, c] - kth) > rtol * kth for c in diff):
                return {"queries": len(qsel), "ok": False, "failed_queries": [int(qsel[j])],
                        "reason": "probe set differs beyond a near tie"}
    D, I = oracle_shard_topk(cfg, st, qsel, gpu_probes)
    if comm.world > 1:
        Ds, Is = comm.allgather(D), comm.allgather(I)
        D, I = topk.merge(list(Ds), list(Is), cfg.topk)
    bad, worst, swaps = [], 0.0, 0
    for j, q in enumerate(qsel):
        g_d, g_i = gd[j].astype(np.float64), gi[j].astype(np.int64)
        nv = int((I[j] >= 0).sum())
        if int((g_i >= 0).sum()) != nv or len(np.unique(g_i[:nv])) != nv:
            bad.append(int(q))
            continue
        ref = D[j][:nv]
        err = np.abs(g_d[:nv] - ref) / np.maximum(ref, 1e-30)
        worst = max(worst, float(err.max()) if nv else 0.0)
        if nv and err.max() > rtol:
            bad.append(int(q))
            continue
        mism = g_i[:nv] != I[j][:nv]
        swaps += int(mism.sum())
        if mism.any():   # an id may differ only among distances tied within the tolerance
            pos = {int(i): p for p, i in enumerate(I[j][:nv])}
            for p in np.flatnonzero(mism):
                other = pos.get(int(g_i[p]))
                if other is None:   # GPU id outside the oracle top-k: its distance must tie the k-th
                    if abs(g_d[p] - ref[-1]) > rtol * max(ref[-1], 1e-30):
                        bad.append(int(q))
                        break
                elif abs(ref[other] - ref[p]) > rtol * max(ref[p], 1e-30):
                    bad.append(int(q))
                    break
    return {"queries": len(qsel), "max_rel_err": worst, "tolerance_id_swaps": swaps, "probe_tie_swaps": probe_swaps,
            "failed_queries": bad, "ok": not bad,
            "protocol": "fp32 distance within 1e-5 rel of the fp64 oracle; ids equal up to swaps among "
                        "distances tied within 1e-5 (DESIGN.md 3.C)"}


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
    comm = Comm(rank, world, dev)
    cfg = synth.CONFIGS[args.config]
    mode = shard_mode(cfg, args, world)
    Q, k = cfg.Q, cfg.topk
    full = (k == 0)
    ivf = bool(cfg.ivf_nlist)
    if full and mode in ("db", "lists"):
        raise SystemExit("full output (c1) cannot be database-sharded: use --shard queries")
    backend = CudaBackend(dev)
    st = prepare(cfg, {}, backend, comm, mode)
    t_b = time.time()
    ix = build_index(cfg, st)
    torch.cuda.synchronize()
    build_s = time.time() - t_b
    log(f"[rank {rank}] index built in {build_s:.2f}s (GPU sort + group, host trees over the distinct codes)")
    stats = ix.stats() if ix is not None else []
    kk = max(k, 1)
    # this rank's queries
    q_lo, q_hi = (rank * Q // world, (rank + 1) * Q // world) if mode == "queries" else (0, Q)
    Ql = q_hi - q_lo
    qd = torch.from_numpy(st["qx"][q_lo:q_hi]).to(dev)
    cbd = torch.from_numpy(st["cb"]).to(dev)
    dist_out = torch.full((Ql, kk), float("inf"), dtype=torch.float32, device=dev)
    ids_out = torch.full((Ql, kk), -1, dtype=torch.int32, device=dev)
    merged = mode in ("db", "lists")
    if merged:
        gd = torch.empty((world, Q, kk), dtype=torch.float32, device=dev)
        gi = torch.empty((world, Q, kk), dtype=torch.int32, device=dev)
    if full:
        full_out = torch.empty((Ql, cfg.N), dtype=torch.float32, device=dev)

    def local_step(q_in):
        if ix is None:                 # empty shard: contributes (+inf, -1) lists
            return dist_out, ids_out
        if full:
            return ix.et_etree_distances(queries=q_in, codebooks=cbd, out=full_out)
        if ivf:
            d_, i_ = ix.et_ivf_topk(q_in, nprobe=cfg.ivf_nprobe, k=k)
            dist_out.copy_(d_)
            ids_out.copy_(i_)
            return dist_out, ids_out
        return ix.et_etree_topk(k, queries=q_in, codebooks=cbd, out=(dist_out, ids_out))

    def gather_merge():
        dist.all_gather_into_tensor(gd, dist_out)
        dist.all_gather_into_tensor(gi, ids_out)

    def step():
        r = local_step(qd)
        if merged:
            gather_merge()
            return api.et_merge_topk(gd, gi)
        return r

    # query.code pairs per step over all ranks (IVF: sizes of the probed lists;
    # every rank probes all Q queries and scans the probed lists it owns)
    if ivf:
        mine = 0
        if ix is not None:
            _, _, pr = ix.et_ivf_topk(qd, nprobe=cfg.ivf_nprobe, k=k, return_probes=True)
            pcells = pr.cpu().numpy().ravel()
            owner = api.et_shard_lists(st["list_sizes"], world) if world > 1 else np.zeros(cfg.ivf_nlist, np.int32)
            mine = int(st["list_sizes"][pcells[owner[pcells] == rank]].sum())
        pairs = int(comm.allsum(np.array([mine], np.int64))[0])
    else:
        pairs = Q * cfg.N

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

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    evs = [(ev(), ev()) for _ in range(args.steps)]
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
    step_ms_rank = sum(a.elapsed_time(b) for a, b in evs) / args.steps
    step_ms = comm.allmax(step_ms_rank)
    value = pairs / (step_ms / 1e3)

    # per-rank terms (N > 1): local (tables + scan + finalize), all-gather, merge
    terms = None
    if world > 1:
        t4 = [(ev(), ev(), ev(), ev()) for _ in range(args.steps)]
        dist.barrier()
        for a, b, c, d in t4:
            flush.fill_(1.0)
            a.record()
            local_step(qd)
            b.record()
            if merged:
                gather_merge()
                c.record()
                api.et_merge_topk(gd, gi)
            else:
                c.record()
            d.record()
        torch.cuda.synchronize()
        mine = np.array([sum(a.elapsed_time(b) for a, b, _, _ in t4), sum(b.elapsed_time(c) for _, b, c, _ in t4),
                         sum(c.elapsed_time(d) for _, _, c, d in t4)]) / args.steps
        allr = comm.allgather(mine)
        terms = {"local_ms": allr[:, 0].round(5).tolist(), "allgather_ms": allr[:, 1].round(5).tolist(),
                 "merge_ms": allr[:, 2].round(5).tolist(), "step_ms_per_rank":
                 comm.allgather(np.array([step_ms_rank]))[:, 0].round(5).tolist(),
                 "n_local_codes": comm.allgather(np.array([len(st["codes"])], np.int64))[:, 0].tolist(),
                 "nccl_ranks": world,
                 "note": ("tables are rebuilt on every rank (queries broadcast): the replicated table "
                          "build is the Amdahl term of db sharding" if mode == "db" else
                          "queries split across ranks: tables and scans split, no collective" if mode == "queries"
                          else "lists split across ranks (LPT); residual tables built for the owned lists")}

    # same-box naive-ADC arm: the same queries through a flat
    # index of the same codes (one leaf per code, LCP 0: N*M lookups) on the
    # same kernels; the E-Tree/E-Forest step vs this is the paper's comparison
    flat = None
    if (world == 1 and not args.no_flat and not ivf and not full and cfg.M <= 8 and ix is not None
            and cfg.N <= 10_000_000):
        fx = api.Index.et_build_flat(st["codes"], ids=st["ids"])
        fd = torch.empty_like(dist_out)
        fi = torch.empty_like(ids_out)
        for _ in range(2):
            fx.et_etree_topk(k, queries=qd, codebooks=cbd, out=(fd, fi))
        f_evs = [(ev(), ev()) for _ in range(max(3, min(args.steps, 10)))]
        torch.cuda.synchronize()
        for a_, b_ in f_evs:
            flush.fill_(1.0)
            a_.record()
            fx.et_etree_topk(k, queries=qd, codebooks=cbd, out=(fd, fi))
            b_.record()
        torch.cuda.synchronize()
        f_ms = sum(a_.elapsed_time(b_) for a_, b_ in f_evs) / len(f_evs)
        same = bool(torch.equal(fd, dist_out)) if not merged else None
        flat = {"flat_adc_ms": f_ms, "etree_ms": step_ms, "etree_over_flat_time": step_ms / f_ms,
                "speedup_vs_flat_adc": f_ms / step_ms, "flat_lookups_per_query": int(cfg.N * cfg.M),
                "same_topk_distances": same,
                "note": "flat = et_build_flat of the same codes through the same scan kernel "
                        "(naive ADC: every code's M lookups); CUDA events, L2 flushed"}
        del fx

    # per-kernel breakdown: the same steps, library events around each launch
    api.et_timing_reset()
    api.et_timing_enable(True)
    for _ in range(args.steps):
        flush.fill_(1.0)
        step()
    torch.cuda.synchronize()
    kern = {}
    for name in ("fill", "probe", "bucket", "cb_chunks", "scan", "finalize", "luts", "gather"):
        ms, n = api.et_timing_get(name)
        if n:
            kern[name] = ms / n
    api.et_timing_enable(False)
    dom = max(kern, key=kern.get) if kern else None

    # e2e: host (pinned) queries in, results out, copies inside the timed region
    qh = torch.from_numpy(st["qx"][q_lo:q_hi]).pin_memory()
    out_shape = (Ql, cfg.N) if full else ((Q, kk) if merged else (Ql, kk))
    dh = torch.empty(out_shape, dtype=torch.float32).pin_memory()
    ih = torch.empty(out_shape if not full else (1, 1), dtype=torch.int32).pin_memory()
    q_stage = torch.empty_like(qd)
    n_e = max(5, args.steps // 4)

    def serial_once():
        q_stage.copy_(qh, non_blocking=True)
        r = local_step(q_stage)
        if full:
            dh.copy_(r, non_blocking=True)
        else:
            if merged:
                gather_merge()
                md, mi = api.et_merge_topk(gd, gi)
            else:
                md, mi = r
            if rank == 0 or not merged:   # the merged result is read back once (rank 0)
                dh.copy_(md, non_blocking=True)
                ih.copy_(mi, non_blocking=True)

    # the library's host-buffer call (et_etree_topk_host): uploads, search and
    # read-backs pipelined in batches on two copy streams + the compute stream;
    # timed interleaved with the serial one-stream sequence (the host link's
    # copy rate drifts between runs on this pool, so the two see the same link)
    use_host = ix is not None and not full and not ivf and not merged

    def host_once():
        ix.et_etree_topk_host(k, qh, cbd, out=(dh, ih), n_batches=args.host_batches)

    if use_host:
        for _ in range(2):
            host_once()
    e_evs = [(ev(), ev()) for _ in range(n_e)]
    p_evs = [(ev(), ev()) for _ in range(n_e)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    for (a, b), (c, d) in zip(e_evs, p_evs):
        flush.fill_(1.0)
        a.record()
        serial_once()
        b.record()
        if use_host:
            flush.fill_(1.0)
            c.record()
            host_once()
            d.record()
    torch.cuda.synchronize()
    e2e_ms = comm.allmax(sum(a.elapsed_time(b) for a, b in e_evs) / n_e)
    e2e_how = "serial: H2D copy, step, D2H copy on one stream"
    e2e_serial_ms = None
    if use_host:
        if world == 1:   # the host outputs equal the device step's (same queries, same kernels)
            assert torch.equal(dh, dist_out.cpu()) and torch.equal(ih, ids_out.cpu()), "host-buffer call differs"
        e2e_serial_ms = e2e_ms
        e2e_ms = comm.allmax(sum(c.elapsed_time(d) for c, d in p_evs) / n_e)
        e2e_how = (f"et_etree_topk_host: pinned host queries in, host top-k out, "
                   f"{api.et_host_batches(Ql, args.host_batches)} batches pipelined (copies on two copy streams)")
    h2d = int(comm.allsum(np.array([qh.numel() * 4], np.int64))[0])
    d2h_mine = dh.numel() * 4 + (0 if full else ih.numel() * 4) if (rank == 0 or not merged) else 0
    d2h = int(comm.allsum(np.array([d2h_mine], np.int64))[0])

    # parity of sampled queries against the oracle (oracle leg), before printing
    parity = None
    if not args.no_parity:
        rng = np.random.default_rng(17)
        nsamp = args.parity_queries if cfg.N <= 10_000_000 else min(args.parity_queries, 4)
        qsel = np.unique(np.concatenate(([0, Q - 1], rng.choice(Q, min(nsamp, Q), replace=False))))
        if mode == "queries":   # the index is replicated: rank 0 checks its own queries alone
            qsel = qsel[(qsel >= q_lo) & (qsel < q_hi)]
        res = local_step(qd)
        if merged:
            gather_merge()
            res = api.et_merge_topk(gd, gi)
        torch.cuda.synchronize()
        off = q_lo if mode == "queries" else 0
        if full:
            parity = parity_full(cfg, st, res.cpu().numpy()[qsel - off], qsel) if rank == 0 else None
        else:
            gdn, gin = res[0].cpu().numpy()[qsel - off], res[1].cpu().numpy()[qsel - off]
            probes = None
            if ivf:
                if ix is not None:
                    _, _, pr = ix.et_ivf_topk(qd, nprobe=cfg.ivf_nprobe, k=k, return_probes=True)
                    probes = pr.cpu().numpy()[qsel]
                probes = comm.bcast(probes if rank == 0 else np.zeros((len(qsel), cfg.ivf_nprobe), np.int32))
            if mode == "queries":
                parity = parity_check(cfg, st, Comm(0, 1), gdn, gin, qsel, probes) if rank == 0 else None
            else:
                parity = parity_check(cfg, st, comm, gdn, gin, qsel, probes)

    peaks, peak_src = load_peaks()
    if rank == 0:
        if full and kern.get("gather", 0) > kern.get("scan", 0):
            hbm = float(peaks.get("hbm_gbs", 6558.1))
            byts = Ql * cfg.N * 4 + cfg.N * 4
            ach = byts / (kern["gather"] / 1e3) / 1e9
            roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": hbm, "unit": "GB/s",
                    "frac": round(ach / hbm, 4), "traffic": None,
                    "kernel": "gather_full_kernel (Q x N fp32 output write)",
                    "note": "algorithmic bytes = 4*Q*N output + 4*N slot->leaf map"}
            dom_ms = kern["gather"]
        else:
            n_tables = Ql * cfg.ivf_nprobe if ivf else Ql
            lookups = None
            if ivf:
                lookups = stats[0]["lookups"] / max(1, len(st["codes"])) * pairs / world
            roof = roofline(cfg, stats, kern["scan"], peaks, clk.summary()["sm_mhz"], Ql, n_tables, lookups)
            dom_ms = kern["scan"]
        roof["peak_source"] = peak_src
        roof["share_of_step"] = round(dom_ms / sum(kern.values()), 4)
        tr = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tr):
            with open(tr) as f:
                roof["traffic"] = json.load(f).get(args.config, {}).get("scan")
        try:   # launch plan (chunks of <= 32 queries, leaf segments, streams per warp)
            plan_info = None if ivf else ix.et_plan_info(Ql, 0 if full else kk)
        except Exception:   # noqa: BLE001  (an older library without et_plan_info)
            plan_info = None
        wl = (f"{cfg.name}: BASELINE configs[{CFG_INDEX[cfg.name]}]" if cfg.name in CFG_INDEX
              else f"{cfg.name}: diagnostic companion")
        par = {"none": "1 GPU",
               "db": f"db-shard{world}: first-level subtrees (et_shard_bounds), queries broadcast, "
                     f"NCCL all-gather + et_merge_topk",
               "lists": f"ivf-lists{world}: inverted lists by LPT (et_shard_lists), NCCL all-gather + et_merge_topk",
               "queries": f"query-split{world}: index replicated, Q/{world} queries per rank, no collective"}[mode]
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wl, "pairs_per_step": pairs,
                       "N": cfg.N, "d": cfg.d, "M": cfg.M, "K": cfg.K, "Q": Q, "k": k,
                       "forest_split": cfg.forest_split, "parallelism": par, "shard_mode": mode,
                       "l2": f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write)",
                       "index_build_s": round(build_s, 3),
                       "plan": plan_info,
                       "timing": ("CUDA graph replay of one step, CUDA events per step" if world == 1
                                  else "CUDA events per step, max over ranks")},
            "roofline": roof,
            "north_star_roofline": north_star_roofline(cfg, stats, step_ms, peaks, Ql,
                                                       Ql * cfg.ivf_nprobe if ivf else None,
                                                       stats[0]["lookups"] / max(1, len(st["codes"])) * pairs / world
                                                       if ivf else None) if stats else None,
            "kernels_ms": {k_: round(v, 5) for k_, v in kern.items()},
            "dominant_kernel": dom,
            "e2e": {"value": pairs / (e2e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms, "how": e2e_how,
                    "serial_ms_per_step": e2e_serial_ms},
            "gpu_launches": int(launches_per_step * args.steps),
            "clocks": clk.summary(),
            "tree_stats": [{kk_: s[kk_] for kk_ in ("L1", "L2", "total_postfix", "lookups", "paper_bytes")}
                           for s in stats],
        }
        if terms is not None:
            out["per_rank"] = terms
        if flat is not None:
            out["flat_adc"] = flat
        if parity is not None:
            out["parity"] = parity
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(cfg, st)
        if parity is not None and not parity["ok"]:
            out.pop("value")
            print(json.dumps(out), flush=True)
            log("[bench] PARITY FAILURE:", parity)
            if world > 1:
                dist.barrier()
                dist.destroy_process_group()
            sys.exit(3)
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------------------- dry run (CPU plumbing test)

def run_dry(args):
    """The multi-rank plumbing on CPU (gloo): self-launch, distributed
    generation, the first-byte / list exchange, per-shard top-k, the list
    all-gather and merge -- with the compute supplied by the backend module
    named in --dry-run (a test module; no GPU).  Rank 0 prints the merged
    result and the backend's single-process reference for comparison."""
    import importlib
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    if world > 1:
        dist.init_process_group("gloo")
    comm = Comm(rank, world)
    modname, _, attr = args.dry_run.partition(":")
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    be = getattr(importlib.import_module(modname), attr or "Backend")()
    over = dict(N=args.dry_n, Q=args.dry_q, n_train=max(2000, args.dry_n // 10), lloyd_iters=3)
    cfg = synth.scaled(synth.CONFIGS[args.config], **over)
    if cfg.ivf_nlist:
        cfg = synth.scaled(cfg, ivf_nlist=16, n_coarse_train=2000)
        over.update(ivf_nlist=16, n_coarse_train=2000)
    mode = shard_mode(cfg, args, world)
    st = prepare(cfg, over, be, comm, mode)
    D, I = be.topk(cfg, st)
    if mode in ("db", "lists") and world > 1:
        from paper_1509_05186_b200 import shard
        gd, gi = shard.gather_lists(torch.from_numpy(D), torch.from_numpy(I))
        D, I = be.merge(gd.numpy(), gi.numpy(), cfg.topk)
    if rank == 0:
        print(json.dumps({"dry_run": True, "world": world, "mode": mode, "config": cfg.name,
                          "n_local": len(st["codes"]), "dist": np.asarray(D).tolist(),
                          "ids": np.asarray(I).tolist()}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


# --------------------------------------------------------------------------- reference arm

def run_reference(args):
    """The oracle (plain numpy) timed on the host cores on the same workload:
    each step is a bounded sample (one query against all N codes: fp64
    tables, naive ADC, exact top-k).  Rank 0 only."""
    rank, world, local = dist_env()
    if rank != 0:
        return
    from oracle import pq, topk
    cfg = synth.CONFIGS[args.config]
    if cfg.ivf_nlist or cfg.N > 10_000_000:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"oracle reference arm is bounded to N <= 1e7 flat configs ({cfg.name})"}), flush=True)
        return
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
        d = pq.adc(table, codes)
        if cfg.topk:
            kth = np.partition(d[0], cfg.topk - 1)[cfg.topk - 1]
            sel = np.flatnonzero(d[0] <= kth)
            topk.topk(d[:, sel], ids[sel], cfg.topk)

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
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle", **cpu_info(),
                            "sample": f"{per_step_q} query x {cfg.N} codes per step (fp64 tables + naive ADC "
                                      f"+ exact top-k of the k-th-value superset)"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(synth.CONFIGS))
    ap.add_argument("--shard", default="auto", choices=["auto", "db", "queries", "lists"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-flat", action="store_true", help="skip the same-box naive-ADC (flat index) arm")
    ap.add_argument("--parity-queries", type=int, default=16)
    ap.add_argument("--host-batches", type=int, default=0,
                    help="batches of the e2e host-buffer call (0: the library default)")
    ap.add_argument("--dry-run", default=None, help="module[:attr] of a CPU test backend (tests/)")
    ap.add_argument("--dry-n", type=int, default=20_000)
    ap.add_argument("--dry-q", type=int, default=8)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    relaunch_if_needed(args)
    if args.impl == "reference":
        run_reference(args)
    elif args.dry_run:
        run_dry(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
