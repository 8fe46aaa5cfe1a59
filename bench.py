#!/usr/bin/env python
"""Benchmark of the B200 MPSM join (BASELINE.json metric: join input tuples/s
(|R|+|S|) and achieved HBM GB/s fraction).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg2] [--threads T] [--no-cpu-baseline] [--no-e2e]

One step = one complete P-MPSM join through the public API ``run_join``
(sort S into runs, partition/sort R, merge-join with fused COUNT / MAX /
checksum, result read back to the host) over the configuration's synthetic
inputs.  At N=1 the workload is BASELINE.json configs[1] (cfg2: |R|=100M,
|S|=400M FK join, 8 GB of 16-B tuples), which fits one B200; ``--config``
selects any other single-GPU config (cfg1, cfg3m1..m16, cfg4).  Under
torchrun (N>1) the ranks run the distributed engine (NCCL all-to-all of R +
NVLink peer reads of S runs) on BASELINE configs[4] (cfg5, strong scaling)
or configs[3] (cfg4), see distributed.bench_main.

Printed JSON line (rank 0):
  value      whole-job tuples/s, inputs resident in HBM, CUDA-event timed, max
             over ranks
  result     (count, MAX, checksum) of the join, checked against the committed
             golden (the reference's own results) or the independent torch
             checker (tests/torch_check.py) on the same arrays
  e2e        the same through run_join with pinned HOST buffers: H2D of the
             inputs and D2H of the result inside the timed region
  roofline   the radix scatter pass seg::k_scatter[_ws] (the dominant kernel):
             algorithmic bytes (packing pass 16 + 8, record passes 8 + 8 B per
             tuple) / its summed CUDA-event launch time inside the timed region
             vs MEASURED_PEAKS.json hbm_gbs; traffic from the committed ncu
             capture (profiles/traffic_scatter.json)
  phase_roofline / step_roofline  bytes each phase actually moves / its time
  cpu_baseline  the reference package (oracle/_ref, numba, all host threads)
             on the SAME arrays (the full workload), median of 3 joins
``--impl reference`` times the reference's own CPU run_join on the full
workload instead (one join per step).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "join input tuples/s (|R|+|S|) and achieved HBM GB/s fraction at 1/2/4/8 B200"

CONFIGS = {
    # name: (n_r, n_s, kind)
    "cfg1": (1_000_000, 4_000_000, "fk"),
    "cfg2": (100_000_000, 400_000_000, "fk"),
    "cfg3m1": (200_000_000, 200_000_000, "fk"),
    "cfg3m4": (200_000_000, 800_000_000, "fk"),
    "cfg3m8": (200_000_000, 1_600_000_000, "fk"),
    "cfg3m16": (200_000_000, 3_200_000_000, "fk"),
    "cfg4": (400_000_000, 1_600_000_000, "negcorr"),
}
# reference results of the seeded inputs (tests/golden/golden.json)
GOLDEN = {
    "cfg1": (4_000_000, 8_587_739_465, 0x7CDED1377072045D),
    "cfg2": (400_000_000, 8_589_753_492, 0xAA48801BE88FA31B),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_inputs(name: str, seed: int = 0):
    from paper_1207_0145_b200 import datagen
    from paper_1207_0145_b200.core import KeyDomain

    n_r, n_s, kind = CONFIGS[name]
    if kind == "fk":
        return datagen.gen_fk(n_r, n_s, seed)
    dom = KeyDomain(1, 1 << 32)
    r, s = datagen.gen_negcorr(n_r, n_s, dom, seed)
    return r, s, dom


# ------------------------------------------------------------ clocks sampler
class Clocks:
    QUERY = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.window = None  # (t0, t1) wall-clock bounds of the timed region
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")

    def start(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.QUERY}",
                                          "--format=csv,noheader,nounits", "-lms", "20"], stdout=self.fh,
                                         stderr=subprocess.DEVNULL)
        except Exception as exc:  # nvidia-smi missing
            log("clock sampling unavailable:", exc)
            self.proc = None

    def mark(self, t0: float, t1: float) -> None:
        """the timed region; samples outside it are dropped"""
        self.window = (t0, t1)

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.fh.close()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        import datetime

        rows = []
        with open(self.path) as fh:
            for line in fh:
                f = [x.strip() for x in line.split(",")]
                if len(f) < 10:
                    continue
                try:
                    ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                    rows.append((ts, float(f[2]), float(f[3]), f[6:10]))
                except ValueError:
                    continue
        if self.window and rows:
            t0, t1 = self.window
            inside = [r for r in rows if t0 - 0.02 <= r[0] <= t1 + 0.02]
            # a timed region shorter than the sampling period: nearest samples
            rows = inside or sorted(rows, key=lambda r: abs(r[0] - (t0 + t1) / 2))[:2]
        for _, smv, mxv, flags in rows:
            sm.append(smv)
            mx = mxv
            for nm, v in zip(names, flags):
                if v.lower() == "active":
                    reasons.add(nm)
        try:
            os.remove(self.path)
        except OSError:
            pass
        loaded = [x for x in sm if x > 0.5 * (mx or 1)] or sm
        return {"sm_mhz": statistics.median(loaded) if loaded else None, "sm_max_mhz": mx,
                "samples": len(sm), "reasons": sorted(reasons)}


# ------------------------------------------------------------- CPU baseline
def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


class ReferenceCPU:
    """The reference's own CPU path on the host cores: the unmodified package
    installed into oracle/_ref (numba, run_join p-mpsm with threads = all host
    cores, tight KeyDomain), or the C oracle port if it is absent.  Runs on
    the SAME numpy arrays the GPU arm consumes."""

    def __init__(self, r, s, dom):
        self.t = cpu_threads()
        self.n = r.cardinality + s.cardinality
        ref_dir = os.path.join(ROOT, "oracle", "_ref")
        if os.path.isdir(os.path.join(ref_dir, "mpsm")):
            sys.path.insert(0, ref_dir)
            import mpsm  # the reference package, unmodified

            self.kind = "reference"
            mpsm.warmup()
            rr, ss = mpsm.Relation(r.keys, r.payloads), mpsm.Relation(s.keys, s.payloads)
            cfg = mpsm.JoinConfig(threads=self.t, algorithm="p-mpsm", key_domain=mpsm.KeyDomain(dom.lower, dom.upper))
            self._call = lambda: mpsm.run_join(rr, ss, cfg)
        else:
            from oracle import oracle as orc

            self.kind = "port"
            self._call = lambda: orc.join(r.keys, r.payloads, s.keys, s.payloads, threads=self.t, lower=dom.lower,
                                          upper=dom.upper, parallel=True)

    def step(self):
        """one wall-clock-timed join -> (seconds, (count, max))"""
        t0 = time.perf_counter()
        out = self._call()
        return time.perf_counter() - t0, (out.match_count, out.aggregate_max)

    def describe(self, what: str) -> dict:
        return {"kind": self.kind, "cores": self.t,
                "sample": f"the full workload (the GPU arm's arrays): p-mpsm run_join, threads={self.t}, {what}"}


def cpu_baseline(r, s, dom, reps: int = 3) -> dict:
    ref = ReferenceCPU(r, s, dom)
    ref.step()  # JIT cache / page-in
    times, res = [], None
    for _ in range(reps):
        dt, res = ref.step()
        times.append(dt)
    med = statistics.median(times)
    d = ref.describe(f"median of {reps} wall-clock runs after one warm-up run")
    d.update({"value": ref.n / med, "unit": "tuples/s", "ms_per_step": 1e3 * med,
              "result": {"match_count": res[0], "aggregate_max": res[1]}})
    return d


def config_of(name: str, dom) -> dict:
    """the workload description shared by both arms (same arrays, same join)"""
    n_r, n_s, kind = CONFIGS[name]
    what = "FK equi-join" if kind == "fk" else "negatively correlated 80-20 skew join, 32-bit keys"
    return {"workload": f"{name}: |R|={n_r:,} |S|={n_s:,} {what}, 16-B (u64,u64) tuples",
            "algorithm": "p-mpsm", "key_domain": [dom.lower, dom.upper],
            "generator": "numpy PCG64 seed 0 (datagen.gen_fk / gen_negcorr)",
            "l2": f"inputs {16 * (n_r + n_s) / 1e9:.1f} GB >> 126 MB L2 (no flush needed)"}


def impl_reference(args):
    """--impl reference: the reference's CPU run_join on the full workload,
    one join per step, on rank 0 (other ranks exit without work)."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    if ws > 1:
        return impl_reference_dist(args, ws)
    t_gen = time.perf_counter()
    r, s, dom = make_inputs(args.config)
    log(f"[bench-ref] generated {args.config} in {time.perf_counter() - t_gen:.1f}s")
    ref = ReferenceCPU(r, s, dom)
    res = None
    for _ in range(args.warmup):
        _, res = ref.step()
    times = []
    for _ in range(args.steps):
        dt, res = ref.step()
        times.append(dt)
    total = sum(times)
    val = args.steps * ref.n / total
    golden = GOLDEN.get(args.config)
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tuples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u64", "data": "synthetic (numpy PCG64 seed 0)",
        "config": config_of(args.config, dom),
        "engine": {"impl": f"reference run_join ({ref.kind}, CPU)", "threads": ref.t},
        "result": {"match_count": res[0], "aggregate_max": res[1],
                   "matches_golden": None if golden is None else tuple(res) == golden[:2]},
        "cpu_baseline": dict(ref.describe(f"{args.steps} timed joins after {args.warmup} warm-up joins"),
                             value=val, unit="tuples/s"),
        "e2e": {"value": val, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def impl_reference_dist(args, ws: int):
    """--impl reference under torchrun (N > 1): our arm runs a DIST_CONFIGS
    workload (cfg5 by default) that no single host holds or finishes in
    minutes, so the reference joins a bounded sample of it -- the same
    generator family at 100M x 400M tuples (cfg5 / 16, cfg4 / 4, one GPU's
    share of weak-scaled cfg2) -- one join per step on rank 0's host cores;
    `config` is our arm's, the sample is named in cpu_baseline.sample."""
    from paper_1207_0145_b200 import datagen
    from paper_1207_0145_b200.core import KeyDomain
    from paper_1207_0145_b200.distributed import dist_workload

    name = args.dist_config or "cfg5"
    config, _, n_r, n_s, kind, scaling = dist_workload(name, ws)
    sn_r, sn_s = 100_000_000, 400_000_000
    if os.environ.get("MPSM_BENCH_REF_SAMPLE"):  # "n_r,n_s": a smaller sample (CPU tests of this arm)
        sn_r, sn_s = (int(v) for v in os.environ["MPSM_BENCH_REF_SAMPLE"].split(","))
    t_gen = time.perf_counter()
    if kind == "fk":
        r, s, dom = datagen.gen_fk(sn_r, sn_s, 0)
    else:
        dom = KeyDomain(1, 1 << 32)
        r, s = datagen.gen_negcorr(sn_r, sn_s, dom, 0)
    log(f"[bench-ref] generated the {name} sample in {time.perf_counter() - t_gen:.1f}s")
    ref = ReferenceCPU(r, s, dom)
    res = None
    for _ in range(args.warmup):
        _, res = ref.step()
    times = []
    for _ in range(args.steps):
        dt, res = ref.step()
        times.append(dt)
    total = sum(times)
    val = args.steps * ref.n / total
    sample = (f"a bounded sample of the workload: the same generator at |R|={sn_r:,} |S|={sn_s:,} "
              f"(1/{n_r // sn_r} of {name}'s {n_r + n_s:,} tuples, key domain [{dom.lower}, {dom.upper})), "
              f"p-mpsm run_join, threads={ref.t}, {args.steps} timed joins after {args.warmup} warm-up joins")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "tuples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
        "scaling": scaling, "vs_baseline": None, "dtype": "u64", "data": "synthetic (numpy PCG64 seed 0)",
        "config": config,
        "engine": {"impl": f"reference run_join ({ref.kind}, CPU)", "threads": ref.t},
        "result": {"match_count": res[0], "aggregate_max": res[1], "of": "the sample"},
        "cpu_baseline": {"kind": ref.kind, "cores": ref.t, "sample": sample, "value": val, "unit": "tuples/s"},
        "e2e": {"value": val, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- ours
def expected_result(name: str, rd, sd):
    """(count, max, checksum) the join must produce, and where it comes from:
    the committed golden (the reference's own count/max) when there is one,
    else the independent torch checker (tests/torch_check.py) on the same
    device arrays -- never this package's kernels."""
    import torch

    golden = GOLDEN.get(name)
    if golden is not None:
        return golden, "golden: the reference's run_join count/max, checksum of its materialized pairs"
    from tests import torch_check as tc

    torch.cuda.empty_cache()
    if CONFIGS[name][2] == "fk":
        want = tc.fk_join(rd, sd)
        how = "independent torch FK gather (tests/torch_check.py)"
    else:
        want = tc.general_join(rd, sd)
        how = "independent torch sort + searchsorted join (tests/torch_check.py)"
    torch.cuda.empty_cache()
    return want, how


def impl_ours(args):
    import torch

    ws, rank, local = dist_env()
    # MPSM_BENCH_DIST=1 runs the multi-GPU path at world size 1 (a smoke
    # test of it on a one-GPU box)
    if ws > 1 or (os.environ.get("MPSM_BENCH_DIST") == "1" and "LOCAL_RANK" in os.environ):
        from paper_1207_0145_b200 import distributed

        return distributed.bench_main(args, METRIC, Clocks)

    import paper_1207_0145_b200 as P
    from paper_1207_0145_b200 import _lib
    from paper_1207_0145_b200.core import JoinConfig, Relation

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    P.warmup()
    t_gen = time.perf_counter()
    r, s, dom = make_inputs(args.config)
    n_r, n_s = r.cardinality, s.cardinality
    n_tot = n_r + n_s
    log(f"[bench] generated {args.config}: |R|={n_r:,} |S|={n_s:,} in {time.perf_counter() - t_gen:.1f}s")
    # resident device inputs
    rd = Relation(torch.from_numpy(r.keys).to(dev), torch.from_numpy(r.payloads).to(dev))
    sd = Relation(torch.from_numpy(s.keys).to(dev), torch.from_numpy(s.payloads).to(dev))
    cfg = JoinConfig(threads=args.threads, algorithm="p-mpsm", key_domain=dom)

    clocks = Clocks(local)
    clocks.start()  # sampling runs from before the warm-up; samples are kept for the timed region only
    for _ in range(args.warmup):
        res = P.run_join(rd, sd, cfg)
    torch.cuda.synchronize()
    result = (res.match_count, res.aggregate_max, res.checksum)
    want, how = expected_result(args.config, rd, sd)
    parity = result == tuple(want)
    if not parity:
        log(f"[bench] PARITY FAILURE {result} != {want} ({how})")

    _lib.profile_enable(True)
    l0 = _lib.launch_count()
    torch.cuda.synchronize()
    w0 = time.time()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    phase = {"sort_public": 0.0, "partition": 0.0, "sort_private": 0.0, "join": 0.0, "total": 0.0}
    for _ in range(args.steps):
        res = P.run_join(rd, sd, cfg)
        for k in phase:
            phase[k] += res.phase_timings[k]
    ev1.record()
    torch.cuda.synchronize()
    clocks.mark(w0, time.time())
    launches = _lib.launch_count() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    prof = {k: _lib.profile_read(k) for k in ("seg_scatter", "seg_scatter_sp", "seg_scatter_pp", "seg_count", "merge",
                                              "merge_partition", "dense_check", "dense_tiles", "dense_join",
                                              "radix_histogram")}
    _lib.profile_enable(False)
    clk = clocks.stop()
    value = n_tot / (ms / 1e3)
    timed_ok = (res.match_count, res.aggregate_max, res.checksum) == result

    # roofline of the dominant kernel, the radix scatter pass (seg::k_scatter):
    # algorithmic bytes per tuple = its reads + writes in the layout it runs:
    # pairs 16 + 16; first pass of a packed sort 16 + 8; later packed passes 8 + 8
    wbits = dom.width_bits
    passes = _lib.load().mpsm_sort_pass_count(wbits)
    from paper_1207_0145_b200 import engine as _eng

    packed = _eng.PACK_RECORDS and 1 <= wbits <= 63
    per_tuple = (24 + 16 * (passes - 1)) if packed else 32 * passes
    onesweep_bytes = float(per_tuple) * (n_r + n_s) * args.steps
    os_ms, os_n = prof["seg_scatter"]
    achieved = onesweep_bytes / (os_ms / 1e3) / 1e9 if os_ms > 0 else None
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peaks = json.load(fh)
    except OSError:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)

    # per-phase HBM roofline (the north star asks >= 60 % on the sort and
    # merge-join phases) on the bytes each phase actually moves in this
    # layout: count sweeps 8 B/tuple per pass + the scatter passes; the merge
    # reads every run once (8 B packed records, 16 B pairs); cross-checked
    # with ncu dram__bytes where a capture is committed (profiles/)
    n_pub, n_priv = max(n_r, n_s), min(n_r, n_s)
    sort_b = 8 * passes + per_tuple
    rec_b = 8 if packed else 16
    phase_roof = {}
    for name, nb in (("sort_public", n_pub * sort_b), ("sort_private", n_priv * sort_b),
                     ("join", (n_r + n_s) * rec_b)):
        t = phase[name] / args.steps
        if t > 0:
            phase_roof[name] = {"bytes": nb, "ms": 1e3 * t, "gbs": nb / t / 1e9, "frac": nb / t / 1e9 / peak}
    moved = sum(v["bytes"] for v in phase_roof.values())
    step_roof = {"bytes": moved, "gbs": moved / (ms / 1e3) / 1e9, "frac": moved / (ms / 1e3) / 1e9 / peak,
                 "floor_ms": 1e3 * moved / (peak * 1e9)}
    # the join kernel alone (the dense-run stream on FK inputs, else the
    # merge): the bytes it moves over its summed CUDA-event time
    jk = "dense_join" if prof["dense_join"][0] > 0 else "merge"
    jms = prof[jk][0] / args.steps
    if "join" in phase_roof and jms > 0:
        nb = (n_r + n_s) * rec_b
        phase_roof["join_kernel"] = {"kernel": "k_dense_flat1 / k_dense_flat" if jk == "dense_join" else "k_merge",
                                     "bytes": nb, "ms": jms, "gbs": nb / jms / 1e6, "frac": nb / jms / 1e6 / peak}
    mfile = os.path.join(ROOT, "profiles", "traffic_join.json")
    if "join_kernel" in phase_roof and jk == "dense_join" and packed and args.config == "cfg2" and os.path.exists(mfile):
        with open(mfile) as f:
            tj = json.load(f)
        phase_roof["join_kernel"]["ncu_dram_bytes"] = tj.get("dram_bytes_per_launch")
        phase_roof["join_kernel"]["ncu_source"] = "profiles/traffic_join.json"

    e2e = None
    if not args.no_e2e:
        rh = Relation(torch.from_numpy(r.keys).pin_memory(), torch.from_numpy(r.payloads).pin_memory())
        sh = Relation(torch.from_numpy(s.keys).pin_memory(), torch.from_numpy(s.payloads).pin_memory())
        for _ in range(2):  # warm the path (staging slots, thread pool, page-in of the pinned columns)
            P.run_join(rh, sh, cfg)
        k = max(1, min(args.steps, args.e2e_steps))
        torch.cuda.synchronize()
        _lib.load().mpsm_upload_bytes(1)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        step_ms = []  # host wall clock per join (run_join returns after its result read): the spread
        for _ in range(k):
            t0 = time.perf_counter()
            out = P.run_join(rh, sh, cfg)
            step_ms.append(round(1e3 * (time.perf_counter() - t0), 2))
        e1.record()
        torch.cuda.synchronize()
        e_ms = e0.elapsed_time(e1) / k
        ok = (out.match_count, out.aggregate_max, out.checksum) == result
        up = int(_lib.load().mpsm_upload_bytes(1)) // k  # packed uploads (8-16 B/tuple)
        col = 0 if up else 16 * n_tot  # else: the columns were copied as they are
        e2e = {"value": n_tot / (e_ms / 1e3), "unit": "tuples/s", "ms_per_step": e_ms, "steps": k,
               "h2d_bytes_per_step": up + col, "d2h_bytes_per_step": 8 * _lib.PAIR_FIELDS, "result_ok": ok,
               "host_input_bytes_per_step": 16 * n_tot, "step_wall_ms": step_ms,
               "input_path": "host-packed records (csrc/upload.cu)" if up else "column copies"}
        del rh, sh

    del rd, sd
    torch.cuda.empty_cache()
    cpu = None
    if not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(r, s, dom, reps=args.cpu_reps)
        except Exception as exc:
            cpu = {"value": None, "unit": "tuples/s", "cores": cpu_threads(), "kind": "reference",
                   "sample": f"failed: {exc!r}"}

    # DRAM bytes per scatter launch from the committed ncu --set full capture
    # (tools/ncu_traffic.py over one bench step's k_scatter launches)
    traffic = traffic_detail = None
    tfile = os.path.join(ROOT, "profiles", "traffic_scatter.json")
    if packed and args.config == "cfg2" and os.path.exists(tfile):
        with open(tfile) as f:
            tj = json.load(f)
        traffic = tj["dram_bytes_per_launch"]
        traffic_detail = {"unit": "bytes per launch (dram read + write)",
                          "algorithmic_bytes_per_launch": tj["algorithmic_bytes_per_launch"],
                          "ratio": tj["traffic_over_algorithmic"], "source": "profiles/traffic_scatter.json"}

    line = {
        "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u64", "data": "synthetic (numpy PCG64 seed 0, SURVEY 8(d) generators)",
        "config": config_of(args.config, dom),
        "engine": {"impl": "paper_1207_0145_b200 run_join (libmpsm_b200.so, sm_100a)", "threads": args.threads,
                   "parallelism": "single GPU"},
        "result": {"match_count": result[0], "aggregate_max": result[1], "checksum": hex(result[2]),
                   "expected": [want[0], want[1], hex(want[2])], "verified_by": how, "matches": parity,
                   "timed_steps_match": timed_ok},
        "phase_ms": {k: 1e3 * v / args.steps for k, v in phase.items()},
        "roofline": {"bound": "hbm", "kernel": "seg::k_scatter (radix scatter pass)", "achieved": achieved,
                     "peak": peak, "unit": "GB/s", "frac": (achieved / peak) if achieved else None,
                     "traffic": traffic, "traffic_detail": traffic_detail,
                     "algorithmic_bytes_per_tuple_per_sort": per_tuple,
                     "layout": "packed 8-B records" if packed else "(key, payload) pairs", "passes_per_sort": passes,
                     "launches": os_n, "peak_source": "MEASURED_PEAKS.json hbm_gbs" if peaks else "fallback"},
        "phase_roofline": phase_roof,
        "step_roofline": step_roof,
        "kernel_ms_per_step": {k: v[0] / args.steps for k, v in prof.items()},
        "gpu_launches": launches,
        "clocks": clk,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--threads", type=int, default=1, help="logical workers T (JoinConfig.threads)")
    ap.add_argument("--dist-config", default=None, choices=["cfg5", "cfg4", "cfg2"],
                    help="multi-GPU workload (torchrun, N>1): cfg5 (default), cfg4, cfg2 per GPU")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-reps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        impl_reference(args)
    else:
        impl_ours(args)


if __name__ == "__main__":
    main()
