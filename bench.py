"""Benchmark of the join-project hot path on B200 (one JSON line on rank 0).

Default workload (the driver's): BASELINE.json configs[1], "cfg2":
pi_{x,z}(R(x,y) join S(y,z)), R and S 5M distinct int32 tuples each, x,z
uniform on [0,500k), y Zipf(1.0) on [0,200k); output = sorted distinct packed
int64 (x,z) codes, |OUT| = 128,713,977,893 per step (~1 TB of codes, emitted
in x-range chunks).  ``--config`` selects the other BASELINE configs:

  cfg1  two-path self-join, 200k tuples (configs[0])     tuples/s
  cfg2  two-path, 5M + 5M (configs[1], default)           tuples/s
  cfg3  3-way star, 3 x 300k, |OUT| = 5000^3              tuples/s
  cfg4  set-similarity join, 2M pairs, c = 4              pairs/s
  cfg5  batched boolean set intersection, 64M + 64M, 4M   answers/s

One step = the whole device path from HBM-resident inputs (index/CSR in HBM):
for the joins degree split, operand build, heavy product, light merge and
the emission of every sorted output code / pair; for BSI the index build
(heavy-y bitsets + light lists) and the answers of the whole batch.  Every
step ends with its result in HBM; ``e2e`` repeats the measurement through
the public API with host buffers (H2D of the inputs and D2H of the results
inside the timed region).  Multi-GPU (torchrun, one process per GPU, NCCL):
the joins shard contiguous x ranges balanced by witness work with the other
side replicated (NCCL broadcast), BSI replicates the index and shards the
batch; no data-path collective; value = all ranks' units / max rank time.

  python bench.py [--gpus N --steps K --warmup W] [--config cfgN] [--impl reference]
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
REF_DIR = os.path.join(ROOT, "baseline", "_ref")
CFG2_OUT = 128_713_977_893      # |OUT| of cfg2 (pinned by tests/test_gpu_fullsize.py)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


def _args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--plan", default="gpu", help="two-path: gpu | default | d1,d2")
    ap.add_argument("--chunk-rows", type=int, default=16384)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-verify", action="store_true", help="skip the untimed checksum pass")
    ap.add_argument("--no-light-work", action="store_true", help="skip the light-pass byte count (diagnostic)")
    ap.add_argument("--x-limit", type=int, default=0, help="debug: only the first X output rows")
    ap.add_argument("--clock-period-ms", type=int, default=100, help="nvidia-smi sampling period during the steps")
    ap.add_argument("--bsi-form", default="auto", choices=["auto", "lists", "records", "walk"],
                    help="cfg5 device algorithm (bsi.BsiEngine); answers are identical")
    return ap.parse_args(argv)


def _dist():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


# ----------------------------------------------------------------- clocks / timers
class ClockSampler:
    """nvidia-smi clocks and throttle reasons, sampled every `period_ms`.

    Started before the warm-up steps -- nvidia-smi's own start-up (NVML
    initialisation) otherwise lands inside the first timed steps and stalls
    the host thread that issues them (a 37-96 ms stall of the second timed
    step in r2m) -- and each sample is timestamped, so stop() keeps only the
    samples taken inside the timed region [mark(), stop()]."""

    def __init__(self, dev_index: int, period_ms: int = 100):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        self.q, self.dev, self.period = q, dev_index, period_ms
        self.t0 = None
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={dev_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", str(period_ms)],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def mark(self):
        """Start of the timed region."""
        self.t0 = time.time()

    @staticmethod
    def _stamp(txt):
        import datetime
        try:
            return datetime.datetime.strptime(txt.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        t1 = time.time()
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        self.f.seek(0)
        rows = [ln.strip().split(", ") for ln in self.f if ln.strip()]
        os.unlink(self.f.name)
        t0 = self.t0 if self.t0 is not None else 0.0
        inside = [r for r in rows if len(r) >= 10 and (lambda t: t is not None and t0 <= t <= t1)(self._stamp(r[0]))]
        when = f"during the timed steps ({self.period} ms period)"
        if not inside:
            # a timed region shorter than the sampling period: the sample
            # nearest after its start (the GPU is still at its under-load clocks)
            after = [r for r in rows if len(r) >= 10 and (self._stamp(r[0]) or 0.0) >= t0]
            inside = after[:1]
            when = "the first sample after the timed steps began (region shorter than the sampling period)"
        if not inside:
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
                inside = [ln.strip().split(", ") for ln in out.stdout.splitlines() if ln.strip()]
                when = "one sample right after the timed steps (region shorter than the sampling period)"
            except (OSError, subprocess.SubprocessError):
                inside = []
        rows = [r[1:] for r in inside if len(r) >= 10]
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in rows:
            for i, nm in enumerate(names):
                if r[5 + i].strip().lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm), "sampled": when}


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


def _reduce_max_sum(t_local: float, n_local: float, world: int):
    """(max over ranks of t, sum over ranks of n)."""
    if world <= 1:
        return t_local, n_local
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    tm = torch.tensor([t_local], dtype=torch.float64, device=dev)
    dist.all_reduce(tm, op=dist.ReduceOp.MAX)
    ns = torch.tensor([n_local], dtype=torch.float64, device=dev)
    dist.all_reduce(ns, op=dist.ReduceOp.SUM)
    return float(tm.item()), float(ns.item())


def _barrier(world: int):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


# ----------------------------------------------------------------- reference package (baseline/_ref)
def reference_package():
    """The unmodified reference package installed into baseline/_ref (pip
    --target), or None when it is absent on this machine."""
    if not os.path.isdir(os.path.join(REF_DIR, "mmjoin")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import mmjoin.joinproject  # noqa: F401
        import mmjoin.relation  # noqa: F401
        return sys.modules["mmjoin"]
    except Exception:  # noqa: BLE001
        return None


def _ref_rel(name, pairs):
    from mmjoin.relation import Relation
    return Relation.from_raw_pairs(name, pairs)


def ref_two_path_slice(Rraw, Sraw, xs_raw, counts=False, barrier=None, self_join=False):
    """The reference's two_path_join (default plan) on sigma_{x in xs} R and S
    (output = the full output restricted to those x); S is
    pre-filtered to the y values of the slice (the reference's semi-join would
    drop the rest; kept tuples keep their order, so its dictionaries are the
    same).  Set-up untimed; returns (operator seconds, |OUT|)."""
    from mmjoin.joinproject import two_path_join
    from mmjoin.relation import build_indexed, semi_join_reduce
    sel = Rraw[np.isin(Rraw[:, 0], xs_raw)]
    sf = Sraw[np.isin(Sraw[:, 1], np.unique(sel[:, 1]))]
    R, S = semi_join_reduce(_ref_rel("R", sel), _ref_rel("S", sf))
    r, s = build_indexed(R), build_indexed(S)
    if barrier is not None:
        barrier.wait()
    t0 = time.perf_counter()
    res = two_path_join(r, s, want_counts=counts)
    return time.perf_counter() - t0, len(res.codes)


def port_two_path_slice(Rraw, Sraw, xs_raw, barrier=None):
    """The pinned numpy port (oracle/) on the same slice (1 thread)."""
    from threadpoolctl import threadpool_limits

    from oracle import mmjoin_oracle as o
    sel = Rraw[np.isin(Rraw[:, 0], xs_raw)]
    with threadpool_limits(limits=1):
        a, b = o.semi_join_many([o.encode(sel), o.encode(Sraw)])
        if barrier is not None:
            barrier.wait()
        t0 = time.perf_counter()
        res = o.two_path(a, b, None)
        return time.perf_counter() - t0, len(res.codes)


# ----------------------------------------------------------------- workloads
class TwoPath:
    """cfg1 / cfg2: two_path_join projection (joinproject.py:155-225)."""

    unit = "tuples/s"

    def __init__(self, args, rank, world):
        self.args, self.rank, self.world = args, rank, world

    def setup_host(self):
        from paper_2002_12459_b200 import datagen
        from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce
        self.wl = wl = datagen.config(self.args.config)
        if wl.self_join:
            self.r = self.s = build_indexed(Relation.from_raw_pairs("R", wl.relations[0]))
        else:
            R, S = semi_join_reduce(Relation.from_raw_pairs("R", wl.relations[0]),
                                    Relation.from_raw_pairs("S", wl.relations[1]))
            self.r, self.s = build_indexed(R), build_indexed(S)
        self.Rraw = wl.relations[0]
        self.Sraw = wl.relations[0] if wl.self_join else wl.relations[1]

    def plan(self):
        from paper_2002_12459_b200.optimizer import PARTITIONED, ThresholdPlan, default_plan, gpu_plan
        a = self.args.plan
        if a == "gpu":
            return gpu_plan(self.r, self.s)
        if a == "default":
            return default_plan(self.r, self.s)
        d1, d2 = (int(v) for v in a.split(","))
        return ThresholdPlan(PARTITIONED, d1, d2)

    def setup(self):
        from paper_2002_12459_b200.device import Workspace, device_relation
        from paper_2002_12459_b200.optimizer import FULL_JOIN
        from paper_2002_12459_b200.shard import shard_of
        self.setup_host()
        r, s = self.r, self.s
        self.p = self.plan()
        self.x_lo, self.x_hi = shard_of(r, s, self.rank, self.world)
        if self.args.x_limit:
            self.x_hi = min(self.x_hi, self.x_lo + self.args.x_limit)
        self.dr = device_relation(r)
        if s is r:
            self.ds = self.dr
        elif self.world > 1:
            # S replicated from rank 0 over NVLink (NCCL broadcast of its CSR)
            from paper_2002_12459_b200.shard import replicate_relation
            self.ds = replicate_relation(device_relation(s) if self.rank == 0 else None, 0)
        else:
            self.ds = device_relation(s)
        p = self.p
        self.d1, self.d2 = (p.delta1, p.delta2) if p.strategy != FULL_JOIN else (max(r.n, s.n),) * 2
        self.ws = Workspace()

    def engine(self):
        from paper_2002_12459_b200.engine import TwoPathEngine
        return TwoPathEngine(self.dr, self.ds, self.p.strategy, self.d1, self.d2, False,
                             chunk_rows=self.args.chunk_rows, ws=self.ws,
                             host_left_deg_r=self.r.left_deg, host_left_deg_s=self.s.left_deg)

    def step(self, timer=None):
        diag = os.environ.get("MMJ_BENCH_DIAG") and timer is not None
        if diag:
            import torch
            t = [time.perf_counter()]
            m0 = torch.cuda.memory_stats().get("num_device_alloc", 0)
        eng = self.engine()
        self.eng = eng
        eng.timer = timer
        if diag:
            t.append(time.perf_counter())
        eng.prepare()
        if diag:
            t.append(time.perf_counter())
        for a, b in eng.chunk_bounds(self.x_lo, self.x_hi):
            eng.run_chunk(a, b, sync=False)
        if diag:
            t.append(time.perf_counter())
            self.diag = getattr(self, "diag", []) + [
                {"engine_ms": round(1e3 * (t[1] - t[0]), 3), "prepare_ms": round(1e3 * (t[2] - t[1]), 3),
                 "chunks_ms": round(1e3 * (t[3] - t[2]), 3),
                 "cuda_mallocs": torch.cuda.memory_stats().get("num_device_alloc", 0) - m0}]
        return eng

    def units(self, eng):
        self.stats = eng.finish()
        return self.stats.out_size

    def verify(self):
        """Untimed pass of the exact timed configuration with the order-
        sensitive checksum (mmj_code_checksum) of every chunk's codes."""
        import torch

        from paper_2002_12459_b200 import _native as nat
        eng = self.engine()
        eng.prepare()
        acc = torch.zeros(2, dtype=torch.int64, device="cuda")
        base = 0
        sizes = []
        for a, b in eng.chunk_bounds(self.x_lo, self.x_hi):
            ch = eng.run_chunk(a, b, sync=False)
            n = int(ch.total_dev.item())
            nat.call("mmj_code_checksum", nat.ptr(ch.codes), n, base, nat.ptr(acc), nat.stream_handle())
            base += n
            sizes.append(n)
        st = eng.finish()
        from paper_2002_12459_b200.shard import combine_checksums
        s, w = (int(v) & (2 ** 64 - 1) for v in acc.cpu().tolist())
        # whole-job stamp: the rank-order concatenation of every shard's codes
        n_all, s, w = combine_checksums(base, s, w)
        out = {"out": n_all, "sum": s, "wsum": w, "max_chunk": max(sizes) if sizes else 0, "chunk_codes": sizes,
               "light_intermediate": st.light_intermediate, "heavy_pairs": st.heavy_pairs}
        if self.world > 1:
            out["scope"] = f"all {self.world} ranks (rank-order concatenation); statistics rank 0's"
        if self.args.config == "cfg2" and not self.args.x_limit:
            out["out_matches_pinned"] = n_all == CFG2_OUT
        return out

    def report(self, phases, t_step, out_local, int8_peak):
        hbm, hbm_kind = _peaks()
        st = self.stats
        r, s = self.r, self.s
        u = int((np.asarray(r.left_deg)[self.x_lo:self.x_hi] > self.d2).sum())
        w = int((np.asarray(s.left_deg) > self.d2).sum())
        w_mma = 2.0 * u * st.k_heavy * w
        light_work = None
        if not self.args.no_light_work and "merge_emit" in phases:
            light_work = self._light_work()
        info = {}
        for name, t in phases.items():
            d = {"ms": 1e3 * t, "share_of_step": t / t_step}
            if name in ("emit", "merge_emit") and t > 0:
                ach = 8.0 * out_local / t / 1e9
                d.update(achieved=ach, unit="GB/s", peak=hbm, frac=ach / hbm, bytes_per_step=8 * out_local)
            if name == "merge_emit" and t > 0:
                d.update(witnesses=st.light_intermediate, witness_rate=st.light_intermediate / t)
                if light_work is not None:
                    b = 8.0 * out_local + light_work["b_light"]
                    d.update(algorithmic_with_light=light_work, achieved_with_light=b / t / 1e9,
                             frac_with_light=b / t / 1e9 / hbm)
            if name == "heavy_mma" and t > 0 and w_mma > 0:
                ops = w_mma / t
                d.update(achieved=ops / 1e12, unit="TOPS(int8)", peak_datasheet=INT8_DATASHEET_OPS / 1e12,
                         frac_datasheet=ops / INT8_DATASHEET_OPS, w_mma_unpadded=w_mma)
                if int8_peak:
                    d.update(peak_measured_cublaslt=int8_peak / 1e12, frac_measured=ops / int8_peak)
            info[name] = d
        dominant = max(phases, key=lambda k: phases[k]) if phases else "merge_emit"
        dom = info.get(dominant, {})
        if dominant == "heavy_mma":
            roof = {"bound": "tensor", "achieved": dom.get("achieved"), "peak": dom.get("peak_datasheet"),
                    "unit": "TOPS", "frac": dom.get("frac_datasheet"), "kernel": "heavy_mma_kernel",
                    "peak_kind": "datasheet int8 dense"}
        else:
            ach = dom.get("achieved")
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": (ach / hbm) if ach else None,
                    "kernel": {"merge_emit": "k_merge_emit", "emit": "k_emit_pf16"}.get(dominant, dominant),
                    "peak_kind": hbm_kind,
                    "algorithmic": "8 B per distinct output code (SURVEY 8(d)) x |OUT| / the kernel's summed "
                                   "CUDA-event time over the step's chunks"}
        roof["traffic"], roof["traffic_detail"] = _ncu_traffic(dominant, self.args.config)
        eng = self.eng
        if eng.heavy_kernel == "or":
            # heavy part inside k_merge_emit: every heavy row ORs its heavy-y
            # bit rows (L2-resident, K x wpr x 4 B) over each of its tiles
            nht = int(((eng.hpos[eng.dr.fwd_idx.long()] >= 0)
                       & (eng.dr.left_deg[eng.dr.fwd_row.long()] > self.d2)).sum().item())
            info["heavy_or"] = {"in_kernel": "k_merge_emit", "heavy_r_tuples": nht,
                                "l2_bytes_per_step": 4 * eng.wpr * nht,
                                "heavy_rows_bytes": 4 * eng.wpr * st.k_heavy,
                                "note": "sparse boolean product R_h x S_h: word i of heavy row x = OR of the "
                                        "heavy-y bit rows of R[x]; replaces the tcgen05 product + chunk bitmap "
                                        "round trip for the projection (tensor-core product still serves "
                                        "counts / star / multiply_counts)"}
        cfg = {"workload": self.wl.description + (" (BASELINE configs[1])" if self.args.config == "cfg2"
                                                   else " (BASELINE configs[0])"),
               "config_name": self.args.config, "out_tuples_per_step": None, "heavy_kernel": eng.heavy_kernel,
               "plan": [self.p.strategy, self.d1, self.d2], "k_heavy": st.k_heavy, "kpad": st.kpad,
               "chunk_rows": self.args.chunk_rows, "chunks": st.chunks,
               "light_intermediate": st.light_intermediate, "heavy_pairs": st.heavy_pairs,
               "l2": "256 MiB L2 flush before every timed step; each step writes ~1 TB of codes"
               if self.args.config == "cfg2" else "256 MiB L2 flush before every timed step"}
        return roof, info, cfg

    def _light_work(self):
        """SURVEY.md 8(d) algorithmic bytes of the light passes over this rank's
        rows: B_light = 8 N_Rl + 4 A_l + 8 D_l (N_Rl R tuples driving a light
        list, A_l the distinct lists' total length, D_l distinct light keys,
        counted on the device by merging the light witnesses alone)."""
        import torch

        from paper_2002_12459_b200 import _native as nat
        from paper_2002_12459_b200.optimizer import PARTITIONED
        eng, r, s = self.eng, self.r, self.s
        x_lo, x_hi = self.x_lo, self.x_hi
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
        a_l = int(sdeg_y[np.unique(ys[full])].sum() + lz_deg[np.unique(ys[~full])].sum())
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
            nat.call("mmj_tile_merge", nat.ptr(bm), 0, a, rows, eng.wpr, eng.dom_z, nat.ptr(dr.fwd_ptr),
                     nat.ptr(dr.fwd_idx), nat.ptr(dr.left_deg), eng.d2, hp, nat.ptr(ds.rev_ptr), nat.ptr(ds.rev_idx),
                     lzp, lzi, 0, 0, nat.ptr(segcnt), nat.ptr(wit), nat.stream_handle())
            d_l += int(segcnt[:nseg].sum(dtype=torch.int64).item())
        return {"n_rl": n_rl, "a_l": a_l, "d_l": d_l, "witnesses_check": int(wit.item()),
                "b_light": 8 * n_rl + 4 * a_l + 8 * d_l}

    # -- CPU legs
    def _slice_xs(self, k, nx):
        lv = np.asarray(self.r.rel.left_values)
        dom = len(lv)
        lo = int(np.linspace(0, max(dom - nx, 0), 97)[k % 97])
        return lv[lo:lo + nx], lo

    def cpu_baseline(self):
        nx = 32 if self.args.config == "cfg2" else 512
        xs, lo = self._slice_xs(48, nx)
        out = {"cores": 1}
        if reference_package() is not None:
            dt, n = ref_two_path_slice(self.Rraw, self.Sraw, xs)
            out.update(value=n / dt, unit=self.unit, kind="reference",
                       sample=f"reference mmjoin.joinproject.two_path_join (baseline/_ref, default plan) on the "
                              f"{nx} dense x values starting at {lo}: {n} distinct tuples in {dt:.2f} s; 1 Python "
                              f"thread (numpy/OpenBLAS default threads for the DGEMM)")
        dtp, npt = port_two_path_slice(self.Rraw, self.Sraw, xs)
        port = {"value": npt / dtp, "unit": self.unit, "kind": "port",
                "sample": f"numpy port (oracle/) of the same slice: {npt} tuples in {dtp:.2f} s, 1 thread"}
        if "value" not in out:
            out.update(port)
        else:
            out["port"] = port
        return out

    def ref_sample_args(self, k, cores):
        nx = 32 if self.args.config == "cfg2" else 512
        return [self._slice_xs(k * cores + j, nx)[0] for j in range(cores)], nx

    def ref_run(self, xs, barrier):
        if reference_package() is not None:
            return ref_two_path_slice(self.Rraw, self.Sraw, xs, barrier=barrier)
        return port_two_path_slice(self.Rraw, self.Sraw, xs, barrier=barrier)

    def ref_describe(self, nx, kind):
        return f"{self.args.config} x-slices of {nx} dense x ({kind} two_path_join, default plan)"

    # -- end to end
    def e2e(self):
        """Same metric through joinproject.two_path_join_chunks(upload="fresh",
        host_buffer=(pinned, pinned)): H2D of the pinned CSR inputs and D2H of
        every chunk's sorted codes inside the timed region."""
        import torch

        from paper_2002_12459_b200.joinproject import two_path_join_chunks
        # 2048-row chunks on one GPU; smaller per rank when N ranks pin their
        # double buffers on one host (2 x the largest chunk's codes each)
        rows = max(256, 2048 // max(self.world, 1))
        # two pinned buffers sized by the largest 2048-row chunk's output
        # (untimed sizing pass), not by the chunk's rows x dom_z cells
        cap = 0
        for part in two_path_join_chunks(self.r, self.s, self.p, chunk_rows=rows, device_output=True,
                                         x_range=(self.x_lo, self.x_hi)):
            cap = max(cap, int(part.codes.numel()))
        host_out = tuple(torch.empty(max(cap, 1), dtype=torch.int64, pin_memory=True) for _ in range(2))
        best, h2d, d2h = None, 0, 0
        for _ in range(self.args.e2e_steps):
            _barrier(self.world)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            nout = 0
            for part in two_path_join_chunks(self.r, self.s, self.p, chunk_rows=rows, host_buffer=host_out,
                                             upload="fresh", x_range=(self.x_lo, self.x_hi)):
                nout += len(part.codes)
                h2d = part.stats["h2d_bytes"]
            torch.cuda.synchronize()
            dt, ntot = _reduce_max_sum(time.perf_counter() - t0, nout, self.world)
            d2h = 8 * nout
            v = ntot / dt
            best = v if best is None else max(best, v)
        return {"value": best, "unit": self.unit, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "steps": self.args.e2e_steps, "pinned_host_bytes": 2 * 8 * cap,
                "api": "joinproject.two_path_join_chunks(upload='fresh', host_buffer=(pinned, pinned))"}


def _ncu_traffic(kernel_phase, config=None):
    """(traffic, detail) of the dominant kernel from the committed `ncu --set
    full` capture (profiles/ncu_traffic.json): the captured launch's own
    dram__bytes_read.sum + dram__bytes_write.sum, unscaled, with that launch's
    algorithmic bytes and their ratio beside it."""
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(tpath):
        return None, None
    with open(tpath) as f:
        t = json.load(f).get(kernel_phase)
    if not isinstance(t, dict) or "dram_bytes_per_launch" not in t:
        return None, None
    if config is not None and t.get("config") not in (None, config):
        return None, None           # the capture is of another config's launch
    detail = {k: t[k] for k in ("kernel", "algorithmic_bytes_per_launch", "traffic_over_algorithmic", "source", "note")
              if k in t}
    return t["dram_bytes_per_launch"], detail


class Star:
    """cfg3: 3-way star join-project (joinproject.py:281-378), composite rows
    (x, z) x w; shards x1 ranges."""

    unit = "tuples/s"

    def __init__(self, args, rank, world):
        self.args, self.rank, self.world = args, rank, world

    def setup_host(self):
        from paper_2002_12459_b200 import datagen
        self.wl = datagen.config("cfg3")

    def setup(self):
        from paper_2002_12459_b200.relation import Relation, build_indexed, semi_join_reduce_many
        from paper_2002_12459_b200.star import StarEngine
        self.setup_host()
        wl = self.wl
        rels = semi_join_reduce_many([Relation.from_raw_pairs(f"R{j}", r) for j, r in enumerate(wl.relations)])
        self.idxs = [build_indexed(x) for x in rels]
        d1 = self.idxs[0].rel.dom_left
        base, extra = divmod(d1, self.world)
        lo = self.rank * base + min(self.rank, extra)
        self.x1 = (lo, lo + base + (1 if self.rank < extra else 0))
        self.eng = StarEngine(self.idxs, False)

    def step(self, timer=None):
        n = [0]

        def sink(a, b, codes, counts):
            n[0] += int(codes.numel())
        self.eng.timer = timer
        self.eng.run(sink, x1_range=self.x1)
        self._n = n[0]
        return None

    def units(self, _):
        return self._n

    def verify(self):
        import torch

        from paper_2002_12459_b200 import _native as nat
        acc = torch.zeros(2, dtype=torch.int64, device="cuda")
        base = [0]

        def sink(a, b, codes, counts):
            n = int(codes.numel())
            nat.call("mmj_code_checksum", nat.ptr(codes), n, base[0], nat.ptr(acc), nat.stream_handle())
            base[0] += n
        self.eng.timer = None
        self.eng.run(sink, x1_range=self.x1)
        from paper_2002_12459_b200.shard import combine_checksums
        s, w = (int(v) & (2 ** 64 - 1) for v in acc.cpu().tolist())
        n, s, w = combine_checksums(base[0], s, w)      # the whole job (rank-order x1 ranges)
        return {"out": n, "sum": s, "wsum": w, "full_cube": n == 5000 ** 3}

    def report(self, phases, t_step, out_local, int8_peak):
        hbm, hbm_kind = _peaks()
        eng = self.eng
        info = {}
        rows = (self.x1[1] - self.x1[0]) * eng.row_per_x1
        for name, t in phases.items():
            d = {"ms": 1e3 * t, "share_of_step": t / t_step}
            if name == "merge_emit" and t > 0:
                ach = 8.0 * out_local / t / 1e9
                d.update(achieved=ach, unit="GB/s", peak=hbm, frac=ach / hbm)
            if name == "heavy_mma" and t > 0 and eng.kh:
                w_mma = 2.0 * rows * eng.kh * eng.dk
                ops = w_mma / t
                d.update(achieved=ops / 1e12, unit="TOPS(int8)", frac_datasheet=ops / INT8_DATASHEET_OPS,
                         w_mma_unpadded=w_mma,
                         note="composite rows (x1,x2) x x3 over heavy y; K = the heavy-y count that minimises the "
                              "modelled step (star.choose_threshold; cfg3 sweep in profiles/r3_star_sweep.txt: "
                              "K = 384 runs this kernel at 0.85 of the datasheet but a 2 ms slower step)")
                if int8_peak:
                    d.update(frac_measured=ops / int8_peak)
            info[name] = d
        dom = info.get("merge_emit", {})
        roof = {"bound": "hbm", "achieved": dom.get("achieved"), "peak": hbm, "unit": "GB/s",
                "frac": dom.get("frac"), "kernel": "k_merge_emit", "peak_kind": hbm_kind,
                "traffic": None, "algorithmic": "8 B per distinct output triple code"}
        cfg = {"workload": self.wl.description + " (BASELINE configs[2])", "config_name": "cfg3",
               "x1_range": list(self.x1), "k_heavy": eng.kh, "light_witnesses": int(eng.wit.item()),
               "l2": "256 MiB L2 flush before every timed step; each step writes 1 TB of codes"}
        return roof, info, cfg

    def _slice(self, k):
        raws = self.wl.relations
        xs = np.unique(raws[0][:, 0])
        return xs[[(k * 977) % len(xs)]]

    def _run_slice(self, x1, ref):
        raws = self.wl.relations
        r0 = raws[0][np.isin(raws[0][:, 0], x1)]
        if ref:
            from mmjoin.joinproject import star_join
            from mmjoin.relation import Relation, build_indexed, semi_join_reduce_many
            rels = semi_join_reduce_many([Relation.from_raw_pairs("R0", r0)] +
                                         [Relation.from_raw_pairs(f"R{j}", raws[j]) for j in (1, 2)])
            idx = [build_indexed(x) for x in rels]
            t0 = time.perf_counter()
            res = star_join(idx, 100, 1)
            return time.perf_counter() - t0, len(res.codes)
        from oracle import mmjoin_oracle as o
        orels = o.semi_join_many([o.encode(r0), o.encode(raws[1]), o.encode(raws[2])])
        t0 = time.perf_counter()
        res = o.star(orels, 100, 1, cap=1 << 40)
        return time.perf_counter() - t0, len(res.codes)

    def cpu_baseline(self):
        ref = reference_package() is not None
        dt, n = self._run_slice(self._slice(1), ref)
        return {"value": n / dt, "unit": self.unit, "cores": 1, "kind": "reference" if ref else "port",
                "sample": f"{'reference mmjoin' if ref else 'numpy port'} star_join(delta1=100, delta2=1) on one "
                          f"x1 value (sigma_x1 R1 with R2, R3 whole): {n} triples in {dt:.2f} s, 1 thread"}

    def ref_sample_args(self, k, cores):
        return [self._slice(k * cores + j) for j in range(cores)], 1

    def ref_run(self, x1, barrier):
        if barrier is not None:
            barrier.wait()
        return self._run_slice(x1, reference_package() is not None)

    def ref_describe(self, nx, kind):
        return f"cfg3 x1-slices of {nx} x1 value ({kind} star_join, delta=(100,1))"

    def e2e(self):
        """star_join through the public entry point from host relations:
        upload, device path, D2H of all 1.25e11 codes into one pinned buffer
        per x1 chunk (streamed), timed end to end."""
        import torch

        from paper_2002_12459_b200 import _native as nat  # noqa: F401
        from paper_2002_12459_b200.star import StarEngine
        cap = self.eng.x1_per_chunk * self.eng.row_per_x1 * self.eng.dk
        host = torch.empty(cap, dtype=torch.int64, pin_memory=True)
        _barrier(self.world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        eng = StarEngine(self.idxs, False)      # uploads the three relations
        n = [0]

        def sink(a, b, codes, counts):
            k = int(codes.numel())
            host[:k].copy_(codes, non_blocking=True)
            torch.cuda.current_stream().synchronize()
            n[0] += k
        eng.run(sink, x1_range=self.x1)
        torch.cuda.synchronize()
        dt, ntot = _reduce_max_sum(time.perf_counter() - t0, n[0], self.world)
        h2d = sum(12 * r.rel.n + 8 * r.rel.dom_left + 8 * r.rel.dom_right for r in self.idxs)
        return {"value": ntot / dt, "unit": self.unit, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": 8 * n[0],
                "steps": 1, "api": "star.StarEngine(relations).run(sink=pinned D2H per x1 chunk)"}


class Ssj:
    """cfg4: ssj_mmjoin (apps.py:65-72): self two-path with exact counts,
    a < b and count >= c fused into the emission; shards x ranges."""

    unit = "pairs/s"

    def __init__(self, args, rank, world):
        self.args, self.rank, self.world = args, rank, world

    def setup_host(self):
        from paper_2002_12459_b200 import datagen
        from paper_2002_12459_b200.apps import SetFamily
        from paper_2002_12459_b200.relation import Relation
        self.pairs = datagen.config("cfg4").relations[0]
        self.fam = SetFamily(Relation.from_raw_pairs("sets", self.pairs))

    def setup(self):
        from paper_2002_12459_b200.apps import _ssj_engine, _ssj_plan
        self.setup_host()
        self.idx = self.fam.indexed
        self.plan = _ssj_plan(self.idx, None, 4)
        from paper_2002_12459_b200.device import Workspace
        self.ws = Workspace()
        self.make = lambda: _ssj_engine(self.idx, 4, self.plan, compact=True, ws=self.ws)
        eng, _ = self.make()
        # triangle work balance: rows a own the cells z > a
        dom = eng.dom_x
        work = np.arange(dom, 0, -1, dtype=np.float64)
        csum = np.concatenate([[0.0], np.cumsum(work)])
        cuts = [0] + [int(np.searchsorted(csum, csum[-1] * k / self.world)) for k in range(1, self.world)] + [dom]
        self.xr = (cuts[self.rank], cuts[self.rank + 1])

    def step(self, timer=None):
        eng, decode = self.make()
        eng.timer = timer
        n = [0]

        def sink(ch):
            decode(ch.codes)
            n[0] += ch.n
        eng.run(sink, self.xr[0], self.xr[1])
        self.eng = eng
        self._n = n[0]
        return eng

    def units(self, eng):
        self.stats = eng.stats
        return self._n

    def verify(self):
        import torch

        from paper_2002_12459_b200 import _native as nat
        eng, decode = self.make()
        acc = torch.zeros(2, dtype=torch.int64, device="cuda")
        acc2 = torch.zeros(2, dtype=torch.int64, device="cuda")
        base = [0]

        def sink(ch):
            codes = decode(ch.codes)
            nat.call("mmj_code_checksum", nat.ptr(codes), ch.n, base[0], nat.ptr(acc), nat.stream_handle())
            cnt = ch.counts.to(torch.int64)
            nat.call("mmj_code_checksum", nat.ptr(cnt), ch.n, base[0], nat.ptr(acc2), nat.stream_handle())
            base[0] += ch.n
        eng.run(sink, self.xr[0], self.xr[1])
        from paper_2002_12459_b200.shard import combine_checksums
        s, w = (int(v) & (2 ** 64 - 1) for v in acc.cpu().tolist())
        cs, cw = (int(v) & (2 ** 64 - 1) for v in acc2.cpu().tolist())
        n, s, w = combine_checksums(base[0], s, w)      # the whole job (rank-order row ranges)
        _, cs, cw = combine_checksums(base[0], cs, cw)
        return {"out": n, "sum": s, "wsum": w, "count_sum": cs, "count_wsum": cw}

    def report(self, phases, t_step, out_local, int8_peak):
        hbm, hbm_kind = _peaks()
        eng = self.eng
        info = {}
        for name, t in phases.items():
            d = {"ms": 1e3 * t, "share_of_step": t / t_step}
            if name == "heavy_mma" and t > 0 and eng.kpad:
                lo, hi = self.xr
                # SSJ keeps z > x only and the product skips tiles below the
                # diagonal: algorithmic work = the upper-triangle cells of
                # this rank's rows, 2 K ops each (unpadded K)
                cells = float(sum(eng.dom_z - x - 1 for x in range(lo, hi)))
                w_mma = 2.0 * cells * eng.stats.k_heavy
                ops = w_mma / t
                d.update(achieved=ops / 1e12, unit="TOPS(int8)", peak_datasheet=INT8_DATASHEET_OPS / 1e12,
                         frac_datasheet=ops / INT8_DATASHEET_OPS, w_mma_unpadded=w_mma,
                         note="exact counts (COUNT16 epilogue), upper-triangle cells z > x only")
                if int8_peak:
                    d.update(peak_measured_cublaslt=int8_peak / 1e12, frac_measured=ops / int8_peak)
            if name == "emit" and t > 0:
                ach = 12.0 * out_local / t / 1e9
                d.update(achieved=ach, unit="GB/s", peak=hbm, frac=ach / hbm, note="12 B per (code, count) pair")
            info[name] = d
        dominant = max(phases, key=lambda k: phases[k]) if phases else "heavy_mma"
        dom = info.get(dominant, {})
        if dominant == "heavy_mma":
            roof = {"bound": "tensor", "achieved": dom.get("achieved"), "peak": INT8_DATASHEET_OPS / 1e12,
                    "unit": "TOPS", "frac": dom.get("frac_datasheet"), "kernel": "heavy_mma_kernel",
                    "peak_kind": "datasheet int8 dense", "traffic": None}
        else:
            ach = dom.get("achieved")
            roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s",
                    "frac": (ach / hbm) if ach else None, "kernel": dominant, "peak_kind": hbm_kind,
                    "traffic": None}
        cfg = {"workload": "SSJ c=4, 2M (set, element) pairs, 100k sets (BASELINE configs[3])",
               "config_name": "cfg4", "plan": [self.plan.strategy, self.plan.delta1, self.plan.delta2],
               "matrix_rows": eng.dom_x, "x_range": list(self.xr), "k_heavy": eng.stats.k_heavy,
               "chunks": eng.stats.chunks, "l2": "256 MiB L2 flush before every timed step"}
        return roof, info, cfg

    def _sets(self, k, n=64):
        lv = np.asarray(self.fam.relation.left_values)
        lo = int(np.linspace(0, len(lv) - n, 97)[k % 97])
        return lv[lo:lo + n]

    def _run_slice(self, sets, ref, barrier=None):
        sub = self.pairs[np.isin(self.pairs[:, 0], sets)]
        if ref:
            from mmjoin.joinproject import two_path_join
            from mmjoin.relation import build_indexed, semi_join_reduce
            A, B = semi_join_reduce(_ref_rel("A", sub), _ref_rel("B", self.pairs))
            a, b = build_indexed(A), build_indexed(B)
            if barrier is not None:
                barrier.wait()
            t0 = time.perf_counter()
            res = two_path_join(a, b, want_counts=True)
            t = res.tuples()
            ra = np.asarray(A.left_values)[t[:, 0]]
            rb = np.asarray(B.left_values)[t[:, 1]]
            keep = int(((ra < rb) & (res.counts >= 4)).sum())     # apps.py:57-62
            return time.perf_counter() - t0, keep
        from oracle import mmjoin_oracle as o
        A, B = o.semi_join_many([o.encode(sub), o.encode(self.pairs)])
        if barrier is not None:
            barrier.wait()
        t0 = time.perf_counter()
        res = o.two_path(A, B, None, want_counts=True)
        t = res.tuples()
        ra = np.asarray(A.left_values)[t[:, 0]]
        rb = np.asarray(B.left_values)[t[:, 1]]
        keep = int(((ra < rb) & (res.counts >= 4)).sum())
        return time.perf_counter() - t0, keep

    def cpu_baseline(self):
        ref = reference_package() is not None
        dt, n = self._run_slice(self._sets(3), ref)
        return {"value": n / dt, "unit": self.unit, "cores": 1, "kind": "reference" if ref else "port",
                "sample": f"{'reference mmjoin' if ref else 'numpy port'} two_path_join(sigma_A sets, sets, "
                          f"want_counts=True) + the a<b, count>=4 filter (apps.py:57-62) for 64 sets A: {n} pairs "
                          f"in {dt:.2f} s, 1 thread"}

    def ref_sample_args(self, k, cores):
        return [self._sets(k * cores + j) for j in range(cores)], 64

    def ref_run(self, sets, barrier):
        return self._run_slice(sets, reference_package() is not None, barrier)

    def ref_describe(self, n, kind):
        return f"cfg4 slices of {n} sets ({kind} two_path_join with counts + SSJ filter)"

    def e2e(self):
        """ssj_mmjoin_arrays through the public API from the host SetFamily:
        upload, count join, a<b / >= c emission, D2H of (a, b, count)."""
        import torch

        from paper_2002_12459_b200.apps import SetFamily, ssj_mmjoin_arrays
        from paper_2002_12459_b200.relation import Relation
        fam = SetFamily(Relation.from_raw_pairs("sets", self.pairs))     # fresh: nothing cached on the device
        _barrier(self.world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a, b, n = ssj_mmjoin_arrays(fam, 4)
        torch.cuda.synchronize()
        dt, ntot = _reduce_max_sum(time.perf_counter() - t0, len(a), self.world)
        return {"value": ntot / dt, "unit": self.unit, "h2d_bytes_per_step": int(8 * 2 * len(self.pairs)),
                "d2h_bytes_per_step": int(len(a) * 24), "steps": 1,
                "api": "apps.ssj_mmjoin_arrays(SetFamily, 4) (whole family on every rank)"}


class Bsi:
    """cfg5: bsi_answer_batch (apps.py:314-351): per-batch index build (records form only: heavy-y bitsets
    + light lists over the device CSR) + answers; the index is replicated on
    every rank, the batch split into contiguous position slices."""

    unit = "answers/s"

    def __init__(self, args, rank, world):
        self.args, self.rank, self.world = args, rank, world

    def setup_host(self):
        from paper_2002_12459_b200 import datagen
        self.wl = datagen.config("cfg5")

    def setup(self):
        import torch

        from paper_2002_12459_b200.bsi import prepare
        from paper_2002_12459_b200.ingest import from_raw_pairs_device
        from paper_2002_12459_b200.shard import batch_slice
        self.setup_host()
        wl = self.wl
        self.raws = [torch.from_numpy(np.ascontiguousarray(r, dtype=np.int64)) for r in wl.relations]
        self.r = from_raw_pairs_device("R", self.raws[0].pin_memory())
        self.s = from_raw_pairs_device("S", self.raws[1].pin_memory())
        # once per relation pair, outside the timed steps (like the CSR build
        # of the IndexedRelation inputs): shared y space, direct id tables and
        # span tables with heavy-y signatures; timed here and reported
        # (the first call also loads torch's topk / sort kernels: timed twice)
        self.prepare_first_ms = self.prepare_ms = 0.0
        for k in range(2):
            self.r._mmj_bsi_cache = None
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            self.sides = prepare(self.r, self.s)
            torch.cuda.synchronize()
            self.prepare_ms = 1e3 * (time.perf_counter() - t0)
            if k == 0:
                self.prepare_first_ms = self.prepare_ms
        nq = len(wl.batch)
        self.qlo, self.qhi = batch_slice(nq, self.rank, self.world)
        q = wl.batch[self.qlo:self.qhi]
        self.qa = torch.from_numpy(np.ascontiguousarray(q[:, 0])).cuda()
        self.qb = torch.from_numpy(np.ascontiguousarray(q[:, 1])).cuda()
        self.nq = self.qhi - self.qlo
        self.ans = torch.empty(max(self.nq, 1), dtype=torch.int8, device="cuda")

    def step(self, timer=None):
        from paper_2002_12459_b200.bsi import BsiEngine
        sR, sS, dom_y = self.sides
        if timer is not None:
            timer.start("build")
        eng = BsiEngine(sR, sS, dom_y, 256, form=self.args.bsi_form)
        eng.build()
        if timer is not None:
            timer.stop("build")
            timer.start("answer")
        eng.answer(self.qa, self.qb, self.nq, out=self.ans)
        if timer is not None:
            timer.stop("answer")
        self.eng = eng
        return eng

    def units(self, eng):
        return self.nq

    def verify(self):
        """Whole-batch stamp: every rank's slice gathered back into batch
        order (shard.gather_batch_answers), then counts and an order-sensitive
        checksum -- identical for any number of ranks."""
        from paper_2002_12459_b200.shard import gather_batch_answers
        nq_all = len(self.wl.batch)
        a = gather_batch_answers(self.ans[: self.nq], nq_all).cpu().numpy()
        return {"answers": int(len(a)), "true": int((a == 1).sum()), "false": int((a == 0).sum()),
                "none": int((a == -1).sum()),
                "checksum": int((np.arange(1, len(a) + 1, dtype=np.uint64) * (a.astype(np.int64) + 2).astype(np.uint64))
                                .sum(dtype=np.uint64))}

    def report(self, phases, t_step, out_local, int8_peak):
        hbm, hbm_kind = _peaks()
        n_in = int(self.sides[0].n + self.sides[1].n)
        b_bsi = 8.0 * n_in + 9.0 * self.nq
        info = {}
        for name, t in phases.items():
            info[name] = {"ms": 1e3 * t, "share_of_step": t / t_step}
        t_ans = phases.get("answer", 0.0)
        if t_ans > 0:
            info["answer"].update(answers_per_s=self.nq / t_ans, bytes_lower_bound=9.0 * self.nq)
        ach = b_bsi / t_step / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "kernel": "bsi build + answer (whole step)", "peak_kind": hbm_kind,
                "algorithmic": "B_bsi = 8 B per input tuple + 9 B per query (SURVEY 8(d) lower bound) / step time"}
        roof["traffic"], roof["traffic_detail"] = _ncu_traffic("bsi_answer", "cfg5") if self.eng.form == "lists" else (None, None)
        cfg = {"workload": self.wl.description + " (BASELINE configs[4])", "config_name": "cfg5",
               "queries_this_rank": self.nq, "batch_slice": [self.qlo, self.qhi], "heavy_bits": 256,
               "bsi_form": self.eng.form,
               "index": "replicated on every rank; per relation pair and outside the timed steps (bsi.prepare, "
                        "cached on the relation objects): shared y ids, direct id tables, span tables with 32-bit "
                        "heavy-y signatures; per batch and inside the step: nothing to build in the lists form "
                        "(records form: heavy-y split + records)",
               "prepare_ms_once_per_relation_pair": round(self.prepare_ms, 3),
               "prepare_ms_first_call_in_process": round(self.prepare_first_ms, 3),
               "answers_per_s_one_batch_with_prepare": self.nq / (t_step + 1e-3 * self.prepare_ms),
               "span_tables": bool(self.sides[0].span and self.sides[1].span),
               "l2": "256 MiB L2 flush before every timed step"}
        return roof, info, cfg

    def _port(self, k, nq):
        from oracle import mmjoin_oracle as o
        if not hasattr(self, "_orels"):
            self._orels = (o.encode(self.wl.relations[0]), o.encode(self.wl.relations[1]))
        q = self.wl.batch
        lo = (k * nq) % max(len(q) - nq, 1)
        t0 = time.perf_counter()
        a = o.bsi(self._orels[0], self._orels[1], q[lo:lo + nq, 0], q[lo:lo + nq, 1])
        return time.perf_counter() - t0, len(a)

    def cpu_baseline(self):
        dt, n = self._port(0, 200_000)
        return {"value": n / dt, "unit": self.unit, "cores": 1, "kind": "port",
                "sample": f"numpy port (oracle.bsi, vectorised per-query set intersection) on a 200k-query "
                          f"sub-batch, relations encoded untimed: {n} answers in {dt:.2f} s.  The reference's "
                          f"bsi_answer_batch re-encodes and scans all 128M raw pairs in Python per call (minutes "
                          f"and tens of GB per batch), so it is not run here"}

    def ref_sample_args(self, k, cores):
        return [k], 200_000

    def ref_run(self, k, barrier):
        return self._port(k, 200_000)

    def ref_describe(self, n, kind):
        return f"cfg5 sub-batches of {n} queries (numpy port of bsi_answer_batch)"

    def e2e(self):
        """bsi_answer_batch_arrays through the public API from host inputs:
        H2D of both relations' raw pairs (device ingest), index build, the
        batch's H2D, answers and their D2H."""
        import torch

        from paper_2002_12459_b200.apps import bsi_answer_batch_arrays
        from paper_2002_12459_b200.ingest import from_raw_pairs_device
        pin = [t.pin_memory() for t in self.raws]
        q = self.wl.batch[self.qlo:self.qhi]
        qa = torch.from_numpy(np.ascontiguousarray(q[:, 0])).pin_memory()
        qb = torch.from_numpy(np.ascontiguousarray(q[:, 1])).pin_memory()
        _barrier(self.world)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = from_raw_pairs_device("R", pin[0])
        s = from_raw_pairs_device("S", pin[1])
        ans = bsi_answer_batch_arrays(r, s, qa.numpy(), qb.numpy())
        torch.cuda.synchronize()
        dt, ntot = _reduce_max_sum(time.perf_counter() - t0, len(ans), self.world)
        h2d = sum(int(t.numel()) * 8 for t in pin) + 16 * len(q)
        return {"value": ntot / dt, "unit": self.unit, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": len(ans),
                "steps": 1, "api": "ingest.from_raw_pairs_device(raw pairs) x2 + apps.bsi_answer_batch_arrays"}


WORKLOADS = {"cfg1": TwoPath, "cfg2": TwoPath, "cfg3": Star, "cfg4": Ssj, "cfg5": Bsi}


# ----------------------------------------------------------------- reference arm
_REF = {}


def _ref_worker(arg):
    return _REF["wl"].ref_run(arg, _REF["barrier"])


def run_reference(args):
    """The reference's CPU implementation of the path on every host core:
    each step runs one bounded slice per core in parallel single-threaded
    worker processes (their timed operators start together); step time = the
    slowest worker, throughput = all slices' units / that.  The reference
    package itself (baseline/_ref) when installed, else the pinned port."""
    import multiprocessing as mp
    rank, world, _ = _dist()
    if rank != 0:
        return
    cores = max(1, len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1))
    wl = WORKLOADS[args.config](args, 0, 1)
    if args.config == "cfg5":
        cores = 1                  # one process (the port vectorises; 2 x 64M pairs per worker would not fit)
    wl.setup_host()
    ref = reference_package() is not None and args.config != "cfg5"
    kind = "reference" if ref else "port"
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    ctx = mp.get_context("fork")
    _REF.update(wl=wl, barrier=ctx.Barrier(cores) if cores > 1 else None)
    tt, nout, size = 0.0, 0, None
    with ctx.Pool(cores) as pool:
        for it in range(args.warmup + args.steps):
            batch, size = wl.ref_sample_args(it, cores)
            res = pool.map(_ref_worker, batch, chunksize=1)
            if it >= args.warmup:
                tt += max(dt for dt, _ in res)
                nout += sum(n for _, n in res)
    v = nout / tt if tt > 0 else 0.0
    line = {
        "metric": METRIC, "impl": "reference", "value": v, "unit": wl.unit, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tt / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": wl.ref_describe(size, kind) + f", {cores} in parallel per step",
                   "config_name": args.config, "package": "baseline/_ref (mmjoin 0.1.0, pip --target)" if ref
                   else "oracle/mmjoin_oracle.py (numpy port)"},
        "cpu_baseline": {"value": v, "unit": wl.unit, "cores": cores, "kind": kind,
                         "sample": f"{args.steps} steps x {cores} slices, {nout} units; {cores} single-threaded "
                                   f"worker processes (OPENBLAS_NUM_THREADS=1)"},
        "e2e": {"value": v, "unit": wl.unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2002_12459_b200 import _native as nat

    rank, world, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    lib = nat.load()
    nat.require_cuda()
    wl = WORKLOADS[args.config](args, rank, world)
    wl.setup()

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    # the cuBLASLt int8 reference runs BEFORE the warm-up steps, so the
    # allocator's cache is in its steady state when the timed steps begin
    int8_peak = _int8_peak_measure() if rank == 0 and args.config != "cfg5" else None
    clocks = ClockSampler(local, args.clock_period_ms)     # started early: see ClockSampler
    for _ in range(args.warmup):
        wl.units(wl.step())
    torch.cuda.synchronize()

    timer = PhaseTimer()
    launches0 = lib.mmj_launch_count()
    times = []
    host_ms = []        # host time to issue each step (diagnostic: the GPU idles when it exceeds the step)
    units = 0
    # no cyclic-GC pause inside a timed step (the step's host thread enqueues
    # every chunk; a collection there leaves the GPU idle): collect between steps
    import gc
    gc_was = gc.isenabled()
    clocks.mark()
    for _ in range(args.steps):
        gc.enable()
        gc.collect()
        gc.disable()
        flush.random_(0, 127)          # 256 MiB write > 126 MB L2
        _barrier(world)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        th = time.perf_counter()
        h = wl.step(timer)
        host_ms.append(round(1e3 * (time.perf_counter() - th), 3))
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
        units = wl.units(h)
        _barrier(world)
    if gc_was:
        gc.enable()
    launches = lib.mmj_launch_count() - launches0
    clk = clocks.stop()
    phases = {k: v / 1e3 / args.steps for k, v in timer.totals().items()}
    t_step = float(np.mean(times))
    t_step_g, units_total = _reduce_max_sum(t_step, float(units), world)
    value = units_total / t_step_g
    roof, info, cfg = wl.report(phases, t_step, units, int8_peak)
    cfg["out_units_per_step"] = int(units_total)
    if "out_tuples_per_step" in cfg:
        cfg["out_tuples_per_step"] = int(units_total)
    cfg["parallelism"] = f"x-range shards x{world}" if args.config != "cfg5" else f"batch slices x{world}"
    check = None if args.no_verify else wl.verify()
    cpu = wl.cpu_baseline() if (rank == 0 and world == 1 and not args.no_cpu_baseline) else None
    e2e = None if args.no_e2e or args.e2e_steps <= 0 else wl.e2e()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": wl.unit, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_step_g, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": cfg, "roofline": roof, "phases": info, "check": check, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches), "clocks": clk, "step_ms": [round(1e3 * t, 3) for t in times],
            "host_issue_ms": host_ms,
            "int8_peak_cublaslt_tops": (int8_peak / 1e12) if int8_peak else None,
            **({"diag": getattr(wl, "diag", None)} if os.environ.get("MMJ_BENCH_DIAG") else {}),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main(argv=None):
    args = _args(argv)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
