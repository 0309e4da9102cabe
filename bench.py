"""Benchmark: distinct output tuples/sec of the two-path join-project hot path.

Workload (BASELINE.json configs[1], "cfg2"): pi_{x,z}(R(x,y) join S(y,z)),
R and S 5M distinct int32 tuples each, x,z uniform on [0,500k), y Zipf(1.0)
on [0,200k), seeds 2/3; output = sorted distinct packed int64 (x,z) codes,
|OUT| ~ 1.26e11 per step (emitted in x-range chunks, ~1 TB of codes).

One step = the whole device path from HBM-resident CSR inputs: degree split,
heavy operand build, tcgen05 heavy product, light expansion, merge/emission
of every chunk's sorted codes into HBM.  Multi-GPU: contiguous dense-x
ranges balanced by witness work, S replicated, no data-path collective (the
one join's output rows are split across ranks: strong scaling); value = all
ranks' |OUT| / max rank time.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "distinct output tuples/sec (2-path, star, sim-join); heavy MMA % INT8 peak"
INT8_DATASHEET_OPS = 4.5e15


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--plan", default="gpu", help="gpu | default | d1,d2")
    ap.add_argument("--chunk-rows", type=int, default=16384)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-light-work", action="store_true", help="skip the light-pass byte count (diagnostic)")
    ap.add_argument("--ref-slice-x", type=int, default=32, help="x values per reference-arm sample")
    ap.add_argument("--x-limit", type=int, default=0, help="debug: only the first X output rows")
    ap.add_argument("--schedule", default="serial", choices=["serial", "mma_ahead", "pipelined"],
                    help="chunk schedule: one stream, heavy product one chunk ahead on a side stream, "
                         "or emission on a side stream")
    return ap.parse_args()


# ----------------------------------------------------------------- workload
def _build(config: str):
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
    wl = datagen.config(config)
    if config not in ("cfg1", "cfg2"):
        raise SystemExit(f"bench.py measures the two-path configs (cfg1, cfg2); got {config}")
    if wl.self_join:
        r = build_indexed(Relation.from_raw_pairs("R", wl.relations[0]))
        return wl, r, r
    R = Relation.from_raw_pairs("R", wl.relations[0])
    S = Relation.from_raw_pairs("S", wl.relations[1])
    R, S = semi_join_reduce(R, S)
    return wl, build_indexed(R), build_indexed(S)


def _plan(args, r, s):
    from paper_2002_12459_b200.optimizer import PARTITIONED, ThresholdPlan, default_plan, gpu_plan
    if args.plan == "gpu":
        return gpu_plan(r, s)
    if args.plan == "default":
        return default_plan(r, s)
    d1, d2 = (int(v) for v in args.plan.split(","))
    return ThresholdPlan(PARTITIONED, d1, d2)


def _light_work(eng, r, s, x_lo: int, x_hi: int):
    """SURVEY.md 8(d) algorithmic bytes of the light passes over rows
    [x_lo, x_hi): B_light = 8 N_Rl + 4 A_l + 8 D_l.

    N_Rl: R tuples that drive a light list (joinproject.py:183-203 restated
    x-side: the full S.rev(y) when y is light or x is light, the light-z part
    of S.rev(y) otherwise); A_l: total length of the distinct lists touched,
    each once; D_l: distinct light (x, z) keys, counted on the device by
    merging the light witnesses alone (k_tile_merge with no heavy bits, outside
    the timed region)."""
    import torch
    from paper_2002_12459_b200 import _native as nat
    from paper_2002_12459_b200.optimizer import PARTITIONED
    t0, t1 = int(r.fwd_indptr[x_lo]), int(r.fwd_indptr[x_hi])
    ys = np.asarray(r.fwd_indices[t0:t1], dtype=np.int64)
    xs = np.repeat(np.arange(x_lo, x_hi, dtype=np.int64), np.diff(r.fwd_indptr[x_lo:x_hi + 1]))
    sdeg_y = np.asarray(s.right_deg, dtype=np.int64)
    if eng.strategy == PARTITIONED and eng.hpos is not None:
        heavy_y = eng.hpos.cpu().numpy()[: len(sdeg_y)] >= 0
        full = (~heavy_y[ys]) | (np.asarray(r.left_deg)[xs] <= eng.d2)
        light_z = np.asarray(s.left_deg) <= eng.d2
        lz_deg = np.add.reduceat(light_z[np.asarray(s.rev_indices)].astype(np.int64),
                                 np.asarray(s.rev_indptr[:-1])) if len(s.rev_indices) else np.zeros(0, np.int64)
        lz_deg = np.where(sdeg_y > 0, lz_deg, 0)
    else:
        full = np.ones(len(ys), bool)
        lz_deg = np.zeros_like(sdeg_y)
    lens = np.where(full, sdeg_y[ys], lz_deg[ys])
    n_rl = int((lens > 0).sum())
    yf = np.unique(ys[full])
    yl = np.unique(ys[~full])
    a_l = int(sdeg_y[yf].sum() + lz_deg[yl].sum())
    # D_l: light-only bitmap per chunk
    d_l = 0
    dr, ds = eng.dr, eng.ds
    hp = nat.ptr(eng.hpos) if eng.strategy == PARTITIONED else 0
    lzp = nat.ptr(eng.lz_ptr) if eng.lz_ptr is not None else 0
    lzi = nat.ptr(eng.lz_idx) if eng.lz_idx is not None else 0
    wit = torch.zeros(1, dtype=torch.int64, device="cuda")
    for a, b in eng.chunk_bounds(x_lo, x_hi):
        rows = b - a
        bm = eng.ws.get("bm", rows * eng.wpr, torch.int32)
        nseg = rows * eng.wpr // 32
        segcnt = eng.ws.get("segcnt", nseg, torch.int32)
        nat.call("mmj_tile_merge", nat.ptr(bm), 0, a, rows, eng.wpr, eng.dom_z,
                 nat.ptr(dr.fwd_ptr), nat.ptr(dr.fwd_idx), nat.ptr(dr.left_deg), eng.d2, hp, nat.ptr(ds.rev_ptr),
                 nat.ptr(ds.rev_idx), lzp, lzi, nat.ptr(segcnt), nat.ptr(wit), nat.stream_handle())
        d_l += int(segcnt[:nseg].sum(dtype=torch.int64).item())
    return {"n_rl": n_rl, "a_l": a_l, "d_l": d_l, "witnesses_check": int(wit.item()),
            "b_light": 8 * n_rl + 4 * a_l + 8 * d_l}


def _shard(r, s, rank: int, world: int):
    """Contiguous dense-x ranges balanced by witness work (shard.py)."""
    from paper_2002_12459_b200.shard import shard_of
    return shard_of(r, s, rank, world)


# ----------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, dev_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={dev_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [ln.strip().split(", ") for ln in self.f if ln.strip()]
        os.unlink(self.f.name)
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            if len(r) < 9:
                continue
            for i, nm in enumerate(names):
                if r[5 + i].strip().lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


class PhaseTimer:
    """CUDA-event brackets around engine phases on the launching stream."""

    def __init__(self):
        import torch
        self.torch = torch
        self.open = {}
        self.done = []

    def start(self, name, stream=None):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(stream)
        self.open[name] = e

    def stop(self, name, stream=None):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(stream)
        self.done.append((name, self.open.pop(name), e))

    def totals(self):
        out = {}
        for name, a, b in self.done:
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out

    def reset(self):
        self.done = []


def _flush_l2(buf):
    buf.random_(0, 127)     # 256 MiB write > 126 MB L2


def _int8_peak_measure():
    """Same-box dense int8 reference: cuBLASLt via torch._int_mm, 8192^3."""
    import torch
    try:
        a = torch.randint(-8, 8, (8192, 8192), dtype=torch.int8, device="cuda")
        b = torch.randint(-8, 8, (8192, 8192), dtype=torch.int8, device="cuda").t()
        for _ in range(3):
            torch._int_mm(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(10):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            torch._int_mm(a, b)
            e.record()
            torch.cuda.synchronize()
            best = min(best, s.elapsed_time(e) / 1e3)
        return 2 * 8192 ** 3 / best
    except Exception:  # noqa: BLE001
        return None


# ----------------------------------------------------------------- CPU legs
def _oracle_slice(wl, r, x_lo: int, nx: int, barrier=None):
    """Oracle two_path on sigma_{x in X'} R (X' = nx consecutive dense x) and S,
    pre-reduced (untimed); returns (elapsed_s, |OUT|).  Single-threaded: BLAS
    pools are limited to one thread so `cores` is exact.  With `barrier`,
    all workers of a parallel step start the timed operator together."""
    from threadpoolctl import threadpool_limits

    from oracle import mmjoin_oracle as o
    lv = np.asarray(r.rel.left_values)
    xs = lv[x_lo:x_lo + nx]
    Rraw = wl.relations[0]
    sel = Rraw[np.isin(Rraw[:, 0], xs)]
    Sraw = wl.relations[0] if wl.self_join else wl.relations[1]
    with threadpool_limits(limits=1):
        a, b = o.semi_join_many([o.encode(sel), o.encode(Sraw)])
        if barrier is not None:
            barrier.wait()
        t0 = time.perf_counter()
        res = o.two_path(a, b, None)
        dt = time.perf_counter() - t0
    return dt, len(res.codes)


_REF = {}


def _ref_worker(args):
    x_lo, nx = args
    return _oracle_slice(_REF["wl"], _REF["r"], x_lo, nx, _REF["barrier"])


def run_reference(args):
    """The reference's CPU implementation of the path (the pinned oracle port)
    on every host core: each step runs one x-slice per core in parallel
    single-threaded worker processes (their timed operators start together);
    step time = the slowest worker, throughput = all slices' tuples / that."""
    import multiprocessing as mp
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2002_12459_b200 import datagen
    from paper_2002_12459_b200.relation import Relation
    wl = datagen.config(args.config)
    R = Relation.from_raw_pairs("R", wl.relations[0])
    dom = R.dom_left

    class _I:   # minimal stand-in exposing rel.left_values for slicing
        rel = R
    nx = args.ref_slice_x
    cores = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    ctx = mp.get_context("fork")
    _REF.update(wl=wl, r=_I, barrier=ctx.Barrier(cores))
    nsl = (args.warmup + args.steps) * cores
    offsets = np.linspace(0, max(dom - nx, 0), nsl + 1).astype(np.int64)
    tt, nout = 0.0, 0
    with ctx.Pool(cores) as pool:
        for it in range(args.warmup + args.steps):
            batch = [(int(offsets[it * cores + k]), nx) for k in range(cores)]
            res = pool.map(_ref_worker, batch, chunksize=1)
            if it >= args.warmup:
                tt += max(dt for dt, _ in res)
                nout += sum(n for _, n in res)
    v = nout / tt if tt > 0 else 0.0
    line = {
        "metric": METRIC, "impl": "reference", "value": v, "unit": "tuples/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tt / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": f"{args.config} x-slices of {nx} dense x (two_path_join, default plan), "
                               f"{cores} in parallel per step", "config_name": args.config},
        "cpu_baseline": {"value": v, "unit": "tuples/s", "cores": cores, "kind": "port",
                         "sample": f"{args.steps} steps x {cores} x-slices of {nx} consecutive dense x values, "
                                   f"{nout} distinct output tuples; {cores} single-threaded worker processes"},
        "e2e": {"value": v, "unit": "tuples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2002_12459_b200 import _native as nat
    from paper_2002_12459_b200.device import DeviceRelation, Workspace, device_relation
    from paper_2002_12459_b200.engine import TwoPathEngine
    from paper_2002_12459_b200.optimizer import FULL_JOIN

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = nat.load()
    nat.require_cuda()

    wl, r, s = _build(args.config)
    plan = _plan(args, r, s)
    x_lo, x_hi = _shard(r, s, rank, world)
    if args.x_limit:
        x_hi = min(x_hi, x_lo + args.x_limit)
    dr = device_relation(r)
    if s is r:
        ds = dr
    elif world > 1:
        # S replicated from rank 0 over NVLink (NCCL broadcast of its CSR)
        from paper_2002_12459_b200.shard import replicate_relation
        ds = replicate_relation(device_relation(s) if rank == 0 else None, 0)
    else:
        ds = device_relation(s)
    d1, d2 = (plan.delta1, plan.delta2) if plan.strategy != FULL_JOIN else (max(r.n, s.n),) * 2
    ws = Workspace()

    def make_engine():
        return TwoPathEngine(dr, ds, plan.strategy, d1, d2, False, chunk_rows=args.chunk_rows, ws=ws,
                             host_left_deg_r=r.left_deg, host_left_deg_s=s.left_deg)

    holder = {}

    def step(timer=None):
        eng = make_engine()
        holder["eng"] = eng
        if args.schedule == "serial":
            eng.timer = timer
            eng.prepare()
            for a, b in eng.chunk_bounds(x_lo, x_hi):
                eng.run_chunk(a, b, sync=False)
        elif args.schedule == "mma_ahead":
            eng.run_mma_ahead(x_lo, x_hi, timer=timer)
        else:
            eng.run_pipelined(x_lo, x_hi, timer=timer)
        return eng.finish()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(args.warmup):
        st_w = step()
    torch.cuda.synchronize()
    int8_peak = _int8_peak_measure() if rank == 0 else None

    timer = PhaseTimer()
    clocks = ClockSampler(local)
    launches0 = lib.mmj_launch_count()
    times = []
    stats = None
    for _ in range(args.steps):
        _flush_l2(flush)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        stats = step(timer)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        if world > 1:
            dist.barrier()
    launches = lib.mmj_launch_count() - launches0
    clk = clocks.stop()
    phases = {k: v / 1e3 / args.steps for k, v in timer.totals().items()}
    t_step = float(np.mean(times))
    out_local = stats.out_size
    if world > 1:
        tt = torch.tensor([t_step, float(out_local)], dtype=torch.float64, device="cuda")
        tmax = tt[:1].clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = tt[1:].clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        t_step_g, out_total = float(tmax.item()), int(tsum.item())
    else:
        t_step_g, out_total = t_step, out_local
    value = out_total / t_step_g

    # ---- roofline of the dominant kernel + the heavy-MMA tensor figure
    hbm, hbm_kind = _peaks()
    eng_last = holder["eng"]
    light_work = None
    if not args.no_light_work and ("light_merge" in phases or "merge_emit" in phases):
        light_work = _light_work(eng_last, r, s, x_lo, x_hi)
    u = int((np.asarray(r.left_deg)[x_lo:x_hi] > d2).sum())
    w = int((np.asarray(s.left_deg) > d2).sum())
    v_k = stats.k_heavy
    w_mma = 2.0 * u * v_k * w
    phase_info = {}
    for name, t in phases.items():
        info = {"ms": 1e3 * t, "share_of_step": t / t_step}
        if name in ("emit", "merge_emit") and t > 0:
            ach = 8.0 * out_local / t / 1e9
            info.update(achieved=ach, unit="GB/s", peak=hbm, frac=ach / hbm, bytes_per_step=8 * out_local)
        if name == "merge_emit" and t > 0:
            info.update(witnesses=stats.light_intermediate, witness_rate=stats.light_intermediate / t)
            if light_work is not None:
                b = 8.0 * out_local + light_work["b_light"]
                info.update(algorithmic_with_light=light_work, achieved_with_light=b / t / 1e9,
                            frac_with_light=b / t / 1e9 / hbm,
                            note="one kernel: light merge + segment scan + look-back + emission; achieved counts "
                                 "the 8 B code writes only, *_with_light adds B_light = 8 N_Rl + 4 A_l + 8 D_l")
        if name == "heavy_mma" and t > 0 and w_mma > 0:
            ops = w_mma / t
            info.update(achieved=ops / 1e12, unit="TOPS(int8)", peak_datasheet=INT8_DATASHEET_OPS / 1e12,
                        frac_datasheet=ops / INT8_DATASHEET_OPS, w_mma_unpadded=w_mma,
                        padded_ops=2.0 * (x_hi - x_lo) * stats.kpad * s.rel.dom_left)
            if int8_peak:
                info.update(peak_measured_cublaslt=int8_peak / 1e12, frac_measured=ops / int8_peak)
        if name in ("light", "light_merge") and t > 0:
            info.update(witnesses=stats.light_intermediate, witness_rate=stats.light_intermediate / t)
            if light_work is not None:
                ach = light_work["b_light"] / t / 1e9
                info.update(achieved=ach, unit="GB/s", peak=hbm, frac=ach / hbm, algorithmic=light_work,
                            bitmap_bytes_per_step=2 * 4 * (x_hi - x_lo) * eng_last.wpr,
                            note="B_light = 8 N_Rl + 4 A_l + 8 D_l (SURVEY 8(d)); the merge also reads and "
                                 "writes the chunk bitmap (bitmap_bytes_per_step), which B_light does not credit")
        phase_info[name] = info
    dominant = max(phases, key=lambda k: phases[k]) if phases else "emit"
    # DRAM bytes per launch from the committed ncu --set full capture, scaled
    # to this run's launches by the measured traffic/algorithmic ratio
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            t = json.load(f).get(dominant)
        if isinstance(t, dict) and dominant in ("emit", "merge_emit") and stats.chunks:
            traffic = t["traffic_over_algorithmic"] * 8.0 * out_local / stats.chunks
        elif isinstance(t, dict):
            traffic = t.get("dram_bytes_per_launch")
    dom = phase_info.get(dominant, {})
    if dominant == "heavy_mma":
        roofline = {"bound": "tensor", "achieved": dom.get("achieved"), "peak": dom.get("peak_datasheet"),
                    "unit": "TOPS", "frac": dom.get("frac_datasheet"), "traffic": traffic,
                    "kernel": "heavy_mma_kernel", "peak_kind": "datasheet int8 dense"}
    else:
        kern = {"emit": "k_emit", "merge_emit": "k_merge_emit", "light": "k_light_expand", "light_merge": "k_tile_merge",
                "segments": "tile_scan"}.get(dominant)
        ach = dom.get("achieved")
        roofline = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": (ach / hbm) if ach else None, "traffic": traffic, "kernel": kern,
                    "peak_kind": hbm_kind}

    # ---- CPU baseline (rank 0, N == 1 only)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        nx = 64
        mid = (x_lo + x_hi) // 2
        dt, n = _oracle_slice(wl, r, mid, nx)
        cpu = {"value": n / dt, "unit": "tuples/s", "cores": 1, "kind": "port",
               "sample": f"oracle two_path_join (default plan) on the {nx} dense x values starting at {mid}: "
                         f"{n} distinct tuples in {dt:.2f} s; one thread (BLAS limited to 1)"}

    # ---- end to end through the public API with host buffers
    e2e = None
    if not args.no_e2e and args.e2e_steps > 0:
        e2e = _e2e(args, r, s, plan, x_lo, x_hi, world)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tuples/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_step_g, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": wl.description + " (BASELINE configs[1])", "config_name": args.config,
                       "out_tuples_per_step": out_total, "plan": [plan.strategy, d1, d2],
                       "k_heavy": stats.k_heavy, "kpad": stats.kpad, "chunk_rows": args.chunk_rows, "schedule": args.schedule,
                       "chunks": stats.chunks, "light_intermediate": stats.light_intermediate,
                       "heavy_pairs": stats.heavy_pairs, "parallelism": f"x-range shards x{world}",
                       "l2": "256 MiB L2 flush before every timed step; each step writes ~1 TB of codes"},
            "roofline": roofline, "phases": phase_info, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk,
            "int8_peak_cublaslt_tops": (int8_peak / 1e12) if int8_peak else None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def _e2e(args, r, s, plan, x_lo, x_hi, world):
    """Same metric through the public chunked API with host buffers:
    joinproject.two_path_join_chunks(upload="fresh") H2D-copies the pinned
    CSR inputs, runs the whole device path and D2H-copies every chunk's
    sorted codes into a pinned host buffer, all inside the timed region."""
    import torch
    import torch.distributed as dist

    from paper_2002_12459_b200.joinproject import two_path_join_chunks

    e2e_rows = min(args.chunk_rows, int(os.environ.get("MMJ_E2E_ROWS", "2048")))
    # two pinned buffers: chunk i+1 is computed while chunk i crosses PCIe
    host_out = tuple(torch.empty(e2e_rows * s.rel.dom_left, dtype=torch.int64, pin_memory=True) for _ in range(2))
    best = None
    h2d = d2h = 0
    for _ in range(args.e2e_steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        nout = 0
        for part in two_path_join_chunks(r, s, plan, chunk_rows=e2e_rows, host_buffer=host_out,
                                         upload="fresh", x_range=(x_lo, x_hi)):
            nout += len(part.codes)
            h2d = part.stats["h2d_bytes"]
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt, float(nout)], dtype=torch.float64, device="cuda")
            tm = t[:1].clone()
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            ts = t[1:].clone()
            dist.all_reduce(ts, op=dist.ReduceOp.SUM)
            dt, nout = float(tm.item()), int(ts.item())
        d2h = 8 * nout
        v = nout / dt
        best = v if best is None else max(best, v)
    out = {"value": best, "unit": "tuples/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
           "steps": args.e2e_steps,
           "api": "joinproject.two_path_join_chunks(upload='fresh', host_buffer=(pinned, pinned))"}
    # informational: the same public call with the output consumed on the
    # device (device_output=True, only each chunk's size read back): what a
    # GPU-side consumer of the join sees, inputs still uploaded every step
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nout = 0
    for part in two_path_join_chunks(r, s, plan, chunk_rows=args.chunk_rows, device_output=True, upload="fresh",
                                     x_range=(x_lo, x_hi)):
        nout += int(part.codes.numel())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([dt, float(nout)], dtype=torch.float64, device="cuda")
        tm = t[:1].clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        ts = t[1:].clone()
        dist.all_reduce(ts, op=dist.ReduceOp.SUM)
        dt, nout = float(tm.item()), int(ts.item())
    out["device_output"] = {"value": nout / dt, "unit": "tuples/s", "h2d_bytes_per_step": int(h2d),
                            "d2h_bytes_per_step": 8 * ((x_hi - x_lo) // max(args.chunk_rows, 1) + 1),
                            "api": "joinproject.two_path_join_chunks(upload='fresh', device_output=True)"}
    return out


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
