#!/usr/bin/env python
"""Benchmark of the batched TT contraction hot path (BASELINE.json metric: TT-pair contractions/s per GPU and x8,
and the fraction of the HBM/FP32 roofline).  One JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--config C2|C1|C3|C4|C5|S1|R1|A2] [--impl ours|reference]

A step is one ttc_inner (ttc_contract for C3) call over the rank's whole batch of synthetic pairs, inputs resident
in HBM, followed at N > 1 by the north star's only collective: the NCCL all_gather of the per-pair results
(dist.gather_results), inside the timed region.  Device time is taken with CUDA events on the launching stream and
the max over ranks is reported.

Main line (the driver's BENCH / SCALE value): BASELINE.json configs[1] (C2: 4,096 pairs of N = 8, I = 16, R = 16)
per GPU -- weak scaling, value = pairs of all ranks / max-over-ranks step time.  The default line also carries
"sub" results, each driver-timed in the same run: C1 (one pair, CUDA graph: us per call), C3 (1,024 pairs
tt_contract), C4 (8,192 pairs, R = 64) and C5 (65,536 pairs, heterogeneous ranks) at their full single-GPU batches;
at N > 1, C4 and C5 are strong-scaled (the same global batch split over the ranks by ttc_partition) and
report E_N = T_1 / (N T_N), T_1 measured by rank 0 on the whole batch in the same run.

--gpus N with no WORLD_SIZE in the environment re-launches this script under torch.distributed.run with N ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import ttgen  # noqa: E402

METRIC = "TT-pair contractions/sec per GPU and x8; fraction of HBM/FP32 roofline"
UNIT = "pairs/s"
L2_BYTES = 126 * 1024 * 1024
SUB_CONFIGS = ("C1", "C3", "C4", "C5")
STRONG = ("C4", "C5")


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="C2", choices=sorted(ttgen.CONFIGS))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--pairs", type=int, default=None, help="pairs per rank (default: the config's batch)")
    p.add_argument("--seed", type=int, default=ttgen.DEFAULT_SEED)
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the oracle sample")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-sub", action="store_true", help="main line only (no C1/C3/C4/C5 sub-results)")
    p.add_argument("--example2", action="store_true", help="Example 2 / Fig. 4a: TTCP vs Eq. 8, cases (i)-(iii)")
    p.add_argument("--sub", default=",".join(SUB_CONFIGS), help="comma list of sub-result configs")
    return p.parse_args()


# floats of one pair's output train (uniform-rank contraction workloads): C3 ladder,
# S1 splice (chain X6^T .. X2^T, K Y2, Y3 .. Y6 of rank 8, I = 8)
PAIR_OUT = {"C3": 102976, "S1": 4224}


# ------------------------------------------------------------------------------------------------ helpers
def config_dict(cfg, B, world, seed, extra=None):
    """The `config` object of a line -- the same keys for the repo arm and the reference arm."""
    c = ttgen.CONFIGS[cfg]
    conf = {"workload": cfg, **{k: (list(v) if isinstance(v, tuple) else v) for k, v in c.items() if k != "op"},
            "op": c["op"], "pairs_per_rank": B, "global_pairs": B * world, "seed": seed,
            "parallelism": f"dp{world}"}
    if extra:
        conf.update(extra)
    return conf


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


def flop_peak_tflops(sm_max_mhz: float) -> float:
    """FP32 FFMA peak = SMs x 128 lanes x 2 flop x max SM clock (B200_PROFILING.md unit counts)."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count if torch.cuda.is_available() else 148
    return sms * 128 * 2 * sm_max_mhz * 1e6 / 1e12


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def pair_macs(xr: np.ndarray, yr: np.ndarray, dims) -> np.ndarray:
    """SURVEY.md Appendix B sweep cost per pair (the host cost model of ttc_pair_cost), from the rank rows only."""
    I = np.asarray(dims, np.float64)[None, :]
    R0, R1 = xr[:, :-1].astype(np.float64), xr[:, 1:].astype(np.float64)
    P0, P1 = yr[:, :-1].astype(np.float64), yr[:, 1:].astype(np.float64)
    return (I * np.minimum(R0 * P1 * (P0 + R1), R1 * P0 * (R0 + P1))).sum(axis=1)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (B200_PROFILING.md recipe)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------------------------ CPU legs
def _oracle_pairs(cfg, X, Y, count, nthreads):
    """The oracle (as it stands) on the first `count` pairs of (X, Y) for workload cfg."""
    import oracle
    c = ttgen.CONFIGS[cfg]
    if cfg in PAIR_OUT:
        per = PAIR_OUT[cfg]
        offs = np.arange(count, dtype=np.int64) * per
        if c["op"] == "splice":
            oracle.tt_splice_batch(X, Y, c["x_mode"], c["y_mode"], offs, per * count, nthreads, 0, count)
        else:
            oracle.tt_contract_batch(X, Y, list(c["x_modes"]), list(c["y_modes"]), offs, per * count, nthreads, 0,
                                     count)
    elif c["op"] == "alg2":          # O6: the dense-input TTCP pipeline per pair (numpy)
        from oracle import ttsvd
        shape = ttgen.alg2_shape(cfg)
        n_el = int(np.prod(shape))
        xh, yh = X.cpu().numpy(), Y.cpu().numpy()
        for b in range(count):
            ttsvd.ttcp_dense(xh[b * n_el:(b + 1) * n_el].reshape(shape, order="F"),
                             yh[b * n_el:(b + 1) * n_el].reshape(shape, order="F"), c["x_mode"], c["y_mode"], c["eps"])
    elif c["op"] == "reconstruct":   # O1a per train (a plain loop; the oracle has no batch entry for it)
        for b in range(count):
            oracle.tt_reconstruct(X.train(b))
    else:
        xc = np.ascontiguousarray(X.cores.detach().cpu().numpy(), dtype=np.float32)
        yc = np.ascontiguousarray(Y.cores.detach().cpu().numpy(), dtype=np.float32)
        oracle.tt_inner_batch_np(xc, yc, X, Y, nthreads, 0, count)


def _oracle_name(cfg):
    op = ttgen.CONFIGS[cfg]["op"]
    return {"contract": "O3", "splice": "O5", "reconstruct": "O1a", "alg2": "O6"}.get(op, "O2")


def cpu_oracle_rate(cfg: str, X, Y, target_s: float, nthreads: int = None, one_thread_s: float = 0.0):
    """Time the oracle (as it stands) on a bounded prefix of the pairs, all host cores (and optionally 1 thread)."""
    nthreads = nthreads or len(os.sched_getaffinity(0))

    def run(count, nt):
        t0 = time.perf_counter()
        _oracle_pairs(cfg, X, Y, count, nt)
        return time.perf_counter() - t0

    nb = X.B if hasattr(X, "B") else X.numel() // int(np.prod(ttgen.alg2_shape(cfg)))
    probe = max(1, min(nb, nthreads))
    t = run(probe, nthreads)
    count = int(min(nb, max(probe, probe * target_s / max(t, 1e-6))))
    reps, t = 0, 0.0
    while reps == 0 or (t < target_s and reps < 1000):
        t += run(count, nthreads)
        reps += 1
    cb = {"value": reps * count / t, "unit": UNIT, "cores": nthreads, "kind": "oracle", "cpu_model": cpu_model(),
          "sample": f"{reps} pass(es) over the first {count} of {nb} {cfg} pairs (fp64 oracle {_oracle_name(cfg)}, "
                    + ("numpy, pairs one after another" if ttgen.CONFIGS[cfg]["op"] == "alg2" else "OpenMP over pairs")
                    + f"), {t:.1f} s"}
    if one_thread_s > 0:
        c1 = max(1, min(count, int(count * one_thread_s / max(t / reps * nthreads, 1e-6))))
        t1 = run(c1, 1)
        cb["one_thread"] = {"value": c1 / t1, "sample": f"first {c1} pairs, 1 thread, {t1:.1f} s"}
        cb["parallel_speedup"] = cb["value"] / (c1 / t1)
    return cb, count, t / reps


def run_reference(args, rank, world):
    """--impl reference: the oracle timed as the reference arm (rank 0 only; other ranks exit without work)."""
    if rank != 0:
        return
    cfg = args.config
    B = args.pairs or ttgen.CONFIGS[cfg]["B"]
    if ttgen.CONFIGS[cfg]["op"] == "alg2":
        X, Y = ttgen.dense_pairs(cfg, 0, B, args.seed, "cpu")
    else:
        X, Y = ttgen.config_batch(cfg, "iid", 0, B, args.seed, "cpu")
    steps_budget = 150.0 / max(1, args.steps + args.warmup)
    cb, count, t = cpu_oracle_rate(cfg, X, Y, min(args.cpu_seconds, steps_budget))
    times = []
    for s in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        _oracle_pairs(cfg, X, Y, count, cb["cores"])
        if s >= args.warmup:
            times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = count / (ms / 1e3)
    cb.update(value=value, sample=f"each step: first {count} of {B} {cfg} pairs, fp64 oracle, {cb['cores']} threads")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_dict(cfg, B, world, args.seed),
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------ GPU arm
class Work:
    """One workload on this rank: step() launches it on `stream`; algorithmic bytes / flops per step."""
    pass


def make_work(ttc, cfg, b0, B, seed, dev, stream, ranks=None):
    """Build pairs b0..b0+B-1 of `cfg` on `dev` and the step that runs them (ranks: C5 rank rows, precomputed)."""
    c = ttgen.CONFIGS[cfg]
    w = Work()
    w.cfg, w.B, w.launches = cfg, B, 1
    if c["op"] == "alg2":
        X, Y = ttgen.dense_pairs(cfg, b0, B, seed, dev)
        XD = YD = None
    else:
        X, Y = ttgen.config_batch(cfg, "iid", b0, B, seed, dev)
        XD, YD = ttc.TTDevice.from_batch(X), ttc.TTDevice.from_batch(Y)
    w.X, w.Y, w.XD, w.YD = X, Y, XD, YD
    if cfg == "C3":
        plan = ttc.ttc_contract_plan_create(XD, YD, c["x_modes"], c["y_modes"])
        out = torch.empty(plan.total, dtype=torch.float32, device=dev)
        w.alg_bytes = 4.0 * (X.cores.numel() + Y.cores.numel()) + 4.0 * plan.total
        w.alg_flops = 2.0 * B * 339968  # structure-aware MACs per pair

        def step():
            ttc.ttc_contract(plan, XD, YD, out=out, stream=stream)
        w.kernel = "contract_kernel"
        w.plan = plan
    elif c["op"] == "splice":
        plan = ttc.ttc_splice_plan_create(XD, YD, c["x_mode"], c["y_mode"])
        out = torch.empty(plan.total, dtype=torch.float32, device=dev)
        w.alg_bytes = 4.0 * (X.cores.numel() + Y.cores.numel()) + 4.0 * plan.total
        # K = A_x^T A_y (I R_1 P_1 MACs) and its absorption into Y_2 (R_1 P_1 J_2 P_2 MACs), per pair
        w.alg_flops = 2.0 * B * (c["I"] * c["R"] * c["P"] + c["R"] * c["P"] * c["I"] * c["P"])

        def step():
            ttc.ttc_contract(plan, XD, YD, out=out, stream=stream)
        w.kernel = "splice_kernel"
    elif c["op"] == "alg2":
        # Alg. 2 on dense operands: TT-SVD of X^rho and Y^rho (step 1's permutation folded into the read),
        # K and the splice (steps 4-5), dense reconstruction in Eq. 8 order (steps 5-6)
        shape = ttgen.alg2_shape(cfg)
        Nd = len(shape)
        px = [c["x_mode"]] + [k for k in range(1, Nd + 1) if k != c["x_mode"]]
        py = [c["y_mode"]] + [k for k in range(1, Nd + 1) if k != c["y_mode"]]
        n_in = int(np.prod(shape))
        joint = px == py   # same shape and permutation: one TT-SVD launch sequence over the 2B tensors [X; Y]
        if joint:
            XY = torch.empty(2 * B * n_in, dtype=torch.float32, device=dev)
            XY[:B * n_in].copy_(X)
            XY[B * n_in:].copy_(Y)
            X, Y = XY[:B * n_in], XY[B * n_in:]   # the e2e leg copies the host inputs into these views
            TXY = ttc.ttc_tt_svd(XY, shape, c["eps"], perm=px)
            cap = ttc.ttc_tt_svd_capacity(shape, px)
            rows = TXY.rank_rows()
            offs = np.arange(B, dtype=np.int64) * cap
            TX = ttc.TTDevice(TXY.cores[:B * cap], TXY.dims_np, ranks=rows[:B], offsets=offs)
            TY = ttc.TTDevice(TXY.cores[B * cap:], TXY.dims_np, ranks=rows[B:], offsets=offs)
        else:
            TX = ttc.ttc_tt_svd(X, shape, c["eps"], perm=px)
            TY = ttc.ttc_tt_svd(Y, shape, c["eps"], perm=py)
        plan = ttc.ttc_splice_plan_create(TX, TY, 1, 1)
        rx_dev = torch.from_numpy(TX.rank_rows()).to(dev)
        ry_dev = torch.from_numpy(TY.rank_rows()).to(dev)
        zc = torch.empty(plan.total, dtype=torch.float32, device=dev)
        ZD = ttc.TTDevice(zc, plan.dims, ranks=plan.ranks, offsets=plan.offsets)
        n_out = int(np.prod(plan.dims.astype(np.int64)))
        out = torch.empty(B * n_out, dtype=torch.float32, device=dev)
        rk_x, rk_y = torch.empty_like(rx_dev), torch.empty_like(ry_dev)
        ws_x = torch.empty(max(16, ttc.ttc_tt_svd_workspace(2 * B if joint else B, shape, px)), dtype=torch.uint8,
                           device=dev)
        ws_y = None if joint else torch.empty(max(16, ttc.ttc_tt_svd_workspace(B, shape, py)), dtype=torch.uint8,
                                              device=dev)
        rk_xy = torch.empty((2 * B, len(shape) + 1), dtype=torch.int32, device=dev) if joint else None
        nb_r = ttc.ttc_reconstruct_workspace(ZD, plan.perm)
        ws_r = torch.empty(nb_r, dtype=torch.uint8, device=dev) if nb_r else None
        train_x = int(sum(int(a) * int(i) * int(b2) for a, i, b2 in
                          zip(TX.rank_rows()[0][:-1], TX.dims_np, TX.rank_rows()[0][1:])))
        w.alg_bytes = 4.0 * B * (2 * n_in + 2 * 2 * train_x + 2 * (plan.total // B) + n_out)
        if cfg == "A2":   # cube 20^3: Gram + Jacobi + products of the two SVD steps, K, splice, reconstruction
            R1, I = int(TX.rank_rows()[0][1]), c["I"]
            svd_mac = 2 * (I * I * n_in // I + 2 * I ** 3 * R1 + 12 * (I - 1) * (I // 2) * I * 6)
            w.alg_flops = 2.0 * B * (svd_mac + I * R1 * R1 + R1 * R1 * I * R1 + n_out * R1 + 2 * I * I * R1 * R1)
        else:             # iterative (one-sided Jacobi) TT-SVD: no fixed flop count; the HBM roofline only
            w.alg_flops = 0.0

        def svd():
            if joint:
                ttc.ttc_tt_svd_into(XY, shape, c["eps"], TXY.cores, rk_xy, perm=px, stream=stream, workspace=ws_x)
                return
            ttc.ttc_tt_svd_into(X, shape, c["eps"], TX.cores, rk_x, perm=px, stream=stream, workspace=ws_x)
            ttc.ttc_tt_svd_into(Y, shape, c["eps"], TY.cores, rk_y, perm=py, stream=stream, workspace=ws_y)

        def splice():
            ttc.ttc_contract(plan, TX, TY, out=zc, stream=stream)

        def recon():
            ttc.ttc_reconstruct(ZD, plan.perm, out=out, stream=stream, workspace=ws_r)

        def step():
            svd()
            splice()
            recon()
        w.stages = {"tt_svd_x_and_y": svd, "splice": splice, "reconstruct": recon}
        w.kernel = "alg2 pipeline (ttsvd x2, splice, reconstruct)"
        # ttc_tt_svd is 1 + 2 (N - 1) launches when every Gram side is <= 32 (the warp-Jacobi pipeline) else 1;
        # the reconstruction 1 launch (shared memory) or L - 1 (workspace GEMM chain, L = output order)
        side = max(min(int(np.prod(shape[:n + 1])), int(np.prod(shape[n + 1:]))) for n in range(Nd - 1))
        per_svd = 1 + 2 * (Nd - 1) if side <= 32 else 1
        w.launches = (1 if joint else 2) * per_svd + 1 + (len(plan.dims) - 1 if nb_r else 1)
        w.plan, w.TX = plan, TX
    elif c["op"] == "reconstruct":
        n_el = c["I"] ** c["N"]
        out = torch.empty(B * n_el, dtype=torch.float32, device=dev)
        w.alg_bytes = 4.0 * X.cores.numel() + 4.0 * out.numel()
        h = c["N"] // 2
        build = sum(c["I"] ** j * c["R"] * c["R"] for j in range(2, h + 1)) * 2
        w.alg_flops = 2.0 * B * (build + n_el * c["R"])

        def step():
            ttc.ttc_reconstruct(XD, None, out=out, stream=stream)
        w.kernel = "reconstruct_kernel"
    else:
        out = torch.empty(B, dtype=torch.float32, device=dev)
        mac, byts = ttc.ttc_pair_cost(XD, YD)
        w.alg_bytes = float(byts.sum())
        w.alg_flops = 2.0 * float(mac.sum())
        # heterogeneous pair costs (C5's random ranks): a cost-descending work list, computed once per batch like a
        # plan (host sort of ttc_pair_cost), so the most expensive pairs start first and the tail is short
        order = ttc.ttc_cost_order(XD, YD) if len(set(np.round(mac, 3))) > 1 else None

        def step():
            ttc.ttc_inner(XD, YD, out=out, stream=stream, order=order)
        w.kernel = {"C1": "inner_small_kernel", "C2": "inner_r16_kernel", "C4": "inner_r64tc_kernel",
                    "C5": "inner_ffma_kernel"}.get(cfg, "inner")
    w.step, w.out = step, out
    w.xin = X.cores if hasattr(X, "cores") else X
    w.yin = Y.cores if hasattr(Y, "cores") else Y
    w.working_set = 4.0 * (w.xin.numel() + w.yin.numel()) + 4.0 * out.numel()
    return w


def time_region(fn, stream, dev, steps, warmup, flush_buf, world, barrier=True):
    """W untimed warm-up steps, then K steps each bracketed by CUDA events on `stream` (L2 flushed before every
    step when flush_buf is given), barrier + synchronize on both sides.  Returns per-step ms (this rank)."""
    for _ in range(warmup):
        if flush_buf is not None:
            flush_buf.fill_(1.0)
        fn()
    torch.cuda.synchronize(dev)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    if world > 1 and barrier:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    for k in range(steps):
        if flush_buf is not None:
            flush_buf.fill_(float(k))
        starts[k].record(stream)
        fn()
        ends[k].record(stream)
    torch.cuda.synchronize(dev)
    if world > 1 and barrier:
        dist.barrier()
    return [s.elapsed_time(e) for s, e in zip(starts, ends)]


def max_over_ranks(v: float, dev, world) -> float:
    t = torch.tensor([v], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def roofline_for(w, ms, peaks, peak_kind, cfg, launch_pairs):
    """Roofline object of the dominant kernel: algorithmic bytes (and flops) per launch / CUDA-event duration."""
    achieved_gbs = w.alg_bytes / (ms / 1e3) / 1e9
    fp32_peak = flop_peak_tflops(float(peaks.get("sm_max_mhz", 1965.0)))
    achieved_tf = w.alg_flops / (ms / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            ent = json.load(open(tpath)).get(cfg)
            if isinstance(ent, dict) and ent.get("pairs") == launch_pairs:
                traffic = ent.get("bytes")
        except Exception:
            traffic = None
    hbm = {"bound": "hbm", "achieved": achieved_gbs, "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
           "frac": achieved_gbs / float(peaks["hbm_gbs"]), "traffic": traffic,
           "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs: copy bandwidth)",
           "algorithmic_bytes_per_launch": w.alg_bytes}
    # FP32 arithmetic roofline (north star: "the slower of the sweep's FLOPs at FP32 peak and the core bytes at
    # HBM bandwidth"); the peak is derived from unit counts and clocks, hence "alu".
    alu = {"bound": "alu", "achieved": achieved_tf, "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved_tf / fp32_peak,
           "traffic": traffic, "peak_source": "148 SMs x 128 FP32 lanes x 2 flop x sm_max_mhz (B200_PROFILING.md unit counts)",
           "algorithmic_flops_per_launch": w.alg_flops}
    t_hbm = w.alg_bytes / (peaks["hbm_gbs"] * 1e9)
    t_alu = w.alg_flops / (fp32_peak * 1e12)
    top, other = (hbm, alu) if t_hbm >= t_alu else (alu, hbm)
    r = dict(top)
    r.update({"kernel": w.kernel, "other": {k: v for k, v in other.items() if k != "traffic"},
              "frac_vs_spec_8TBs": achieved_gbs / 8000.0})
    return r


def c1_graph_latency(ttc, dev, seed, reps=200):
    """C1 (one pair): the call captured in a CUDA graph; per-call latency = one replay bracketed by events (median
    of `reps`), and the back-to-back replay rate.  Host validation and the ctypes call are outside the graph."""
    w = make_work(ttc, "C1", 0, 1, seed, dev, None)
    s = torch.cuda.Stream(dev)
    with torch.cuda.stream(s):
        for _ in range(3):
            ttc.ttc_inner(w.XD, w.YD, out=w.out, stream=s)
        torch.cuda.synchronize(dev)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            ttc.ttc_inner(w.XD, w.YD, out=w.out, stream=s)
    torch.cuda.synchronize(dev)
    lat = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(reps):
        with torch.cuda.stream(s):
            e0.record(s)
            g.replay()
            e1.record(s)
        e1.synchronize()
        lat.append(e0.elapsed_time(e1) * 1e3)
    n = 1000
    with torch.cuda.stream(s):
        e0.record(s)
        for _ in range(n):
            g.replay()
        e1.record(s)
    e1.synchronize()
    b2b = e0.elapsed_time(e1) * 1e3 / n
    return {"us_per_call_graph": statistics.median(lat), "us_per_call_p90": float(np.percentile(lat, 90)),
            "us_per_call_back_to_back": b2b, "value": 1e6 / statistics.median(lat), "unit": "calls/s",
            "reps": reps, "kernel": "inner_small_kernel", "roofline": {"bound": "latency", "frac": None,
                                                                         "note": "one pair: launch + DRAM latency"}}


def run_sub(ttc, cfg, args, rank, world, dev, stream, peaks, peak_kind, flush_buf):
    """A driver-timed sub-result for one config at its full single-GPU batch (strong-scaled at N > 1)."""
    import torch.distributed as dist
    c = ttgen.CONFIGS[cfg]
    G = c["B"]
    steps, warm = max(3, min(args.steps, 10)), max(3, min(args.warmup, 3))
    res = {"workload": cfg, "global_pairs": G}
    if cfg == "C1":
        if rank == 0:
            res.update(c1_graph_latency(ttc, dev, args.seed))
        return res
    if world > 1 and cfg in STRONG:
        from paper_2109_00626_b200 import dist as tdist
        if cfg == "C5":
            xr = ttgen.random_ranks(args.seed, ttgen.CFG_ID[cfg], ttgen.SIDE_X, 0, G, c["N"], c["rank_choices"])
            yr = ttgen.random_ranks(args.seed, ttgen.CFG_ID[cfg], ttgen.SIDE_Y, 0, G, c["N"], c["rank_choices"])
            cost = pair_macs(xr, yr, (c["I"],) * c["N"])
        else:
            cost = np.ones(G)
        bounds = ttc.ttc_partition(cost, world)
        lo, hi = int(bounds[rank]), int(bounds[rank + 1])
        w = make_work(ttc, cfg, lo, hi - lo, args.seed, dev, stream)

        def fn():
            w.step()
            tdist.gather_results(w.out, bounds)
        per = time_region(fn, stream, dev, steps, warm, None, world)
        ms_n = max_over_ranks(statistics.median(per), dev, world)
        del w
        torch.cuda.empty_cache()
        # T_1: rank 0 alone runs the whole batch on its GPU (the others wait at the barrier)
        t1 = None
        if rank == 0:
            w1 = make_work(ttc, cfg, 0, G, args.seed, dev, stream)
            t1 = statistics.median(time_region(w1.step, stream, dev, steps, warm, None, 1))
            res["roofline_1gpu"] = roofline_for(w1, t1, peaks, peak_kind, cfg, G)
            del w1
            torch.cuda.empty_cache()
        dist.barrier()
        res.update({"n_gpus": world, "ms_per_step": ms_n, "value": G / (ms_n / 1e3), "unit": UNIT,
                    "scaling": "strong", "timed": "shard kernel + NCCL all_gather of the results (max over ranks)",
                    "shard_pairs": [int(bounds[r + 1] - bounds[r]) for r in range(world)]})
        if rank == 0:
            res.update({"t1_ms": t1, "efficiency": t1 / (world * ms_n)})
        return res
    # world == 1 (or a config that is not strong-scaled): this rank's full batch
    w = make_work(ttc, cfg, rank * G, G, args.seed, dev, stream)
    fb = flush_buf if w.working_set < 2 * L2_BYTES else None
    per = time_region(w.step, stream, dev, steps, warm, fb, world)
    ms = max_over_ranks(statistics.median(per), dev, world)
    res.update({"ms_per_step": ms, "value": G * world / (ms / 1e3), "unit": UNIT,
                "roofline": roofline_for(w, statistics.median(per), peaks, peak_kind, cfg, G),
                "l2": "flushed between steps (2x L2 write)" if fb is not None else "inputs larger than L2",
                "steps": steps, "warmup": warm, "gpu_launches": steps * w.launches})
    if rank == 0 and world == 1 and not args.no_cpu:
        Xh = ttgen.TTBatch(w.X.cores.cpu(), w.X.ranks, w.X.offsets, w.X.dims)
        Yh = ttgen.TTBatch(w.Y.cores.cpu(), w.Y.ranks, w.Y.offsets, w.Y.dims)
        res["cpu_baseline"], _, _ = cpu_oracle_rate(cfg, Xh, Yh, 3.0)
    del w
    torch.cuda.empty_cache()
    return res


def run_example2(ttc, args, dev, stream, peaks, peak_kind, flush_buf):
    """Example 2 (Fig. 4a): X x_1^1 Y of two zero-mean unit-variance Gaussian tensors, cases
    (i) 20^3, (ii) 20 x 20 x 20 x 5, (iii) 20 x 20 x 20 x 5 x 4, "both in the original form via Eq. 8 and through
    the proposed TTCP algorithm" (time including the TT decompositions).  On the GPU: the TTCP pipeline (TT-SVD
    of both operands, K + splice, and the dense reconstruction in Eq. 8 order) and, as the dense-TCP baseline,
    Eq. 8 as one batched fp32 GEMM (cuBLAS through torch.bmm: Z^T = Y_(1)^T X_(1), a plain library GEMM).  On
    the host: the oracle's TTCP (O6, numpy) and Eq. 8 by numpy tensordot on a bounded sample.  The paper prints
    no times for this figure, so there is nothing to compare against but the two arms."""
    torch.backends.cuda.matmul.allow_tf32 = False
    cases = []
    clocks = ClockSampler(dev.index or 0).start()
    for cfg, label in (("A2", "i"), ("A2ii", "ii"), ("A2iii", "iii")):
        c = ttgen.CONFIGS[cfg]
        B = c["B"]
        shape = ttgen.alg2_shape(cfg)
        w = make_work(ttc, cfg, 0, B, args.seed, dev, stream)
        fb = flush_buf if w.working_set < 2 * L2_BYTES else None
        steps, warm = 3, 3
        ms = statistics.median(time_region(w.step, stream, dev, steps, warm, fb, 1))
        stages = {k: statistics.median(time_region(f, stream, dev, steps, warm, fb, 1)) / B
                  for k, f in w.stages.items()}
        # dense-TCP baseline: Eq. 8 as one batched GEMM on the same operands (unfoldings read in place)
        I1 = shape[0]
        rest = int(np.prod(shape[1:]))
        Xt, Yt = w.X.view(B, rest, I1), w.Y.view(B, rest, I1)
        dense = torch.empty((B, rest, rest), dtype=torch.float32, device=dev)

        def eq8():
            torch.bmm(Yt, Xt.transpose(1, 2), out=dense)
        ms_eq8 = statistics.median(time_region(eq8, stream, dev, steps, warm, fb, 1))
        # sanity: the two arms agree on pair 0 (eps = 0: exact TTCP up to rounding)
        n_out = rest * rest
        a0 = w.out[:n_out].view(rest, rest)
        rel = float((a0 - dense[0]).norm() / dense[0].norm())
        case = {"case": label, "workload": cfg, "shape": list(shape), "pairs": B, "eps": c["eps"],
                "ttcp_ms_per_pair": ms / B, "ttcp_stage_ms_per_pair": stages,
                "ttcp_tt_result_ms_per_pair": stages["tt_svd_x_and_y"] + stages["splice"],
                "eq8_gemm_ms_per_pair": ms_eq8 / B, "eq8_over_ttcp": (ms_eq8 / B) / (ms / B),
                "tt_ranks_x": [int(v) for v in w.TX.rank_rows()[0]], "output_entries": n_out,
                "rel_diff_pair0": rel, "gpu_launches_per_step": w.launches,
                "roofline": roofline_for(w, ms, peaks, peak_kind, cfg, B),
                "l2": "flushed between steps (2x L2 write)" if fb is not None else "inputs larger than L2"}
        if not args.no_cpu:
            from oracle import ttsvd
            xh, yh = w.X[:rest * I1].cpu().numpy(), w.Y[:rest * I1].cpu().numpy()
            x0 = xh.astype(np.float64).reshape(shape, order="F")
            y0 = yh.astype(np.float64).reshape(shape, order="F")
            reps = 0
            t0 = time.perf_counter()
            while reps == 0 or (time.perf_counter() - t0 < 3.0 and reps < 50):
                ttsvd.ttcp_dense(x0, y0, 1, 1, c["eps"])
                reps += 1
            t_ttcp = (time.perf_counter() - t0) / reps
            reps2 = 0
            t0 = time.perf_counter()
            while reps2 == 0 or (time.perf_counter() - t0 < 3.0 and reps2 < 50):
                np.tensordot(x0, y0, axes=([0], [0]))
                reps2 += 1
            t_eq8 = (time.perf_counter() - t0) / reps2
            case["cpu"] = {"ttcp_oracle_ms_per_pair": 1e3 * t_ttcp, "eq8_tensordot_ms_per_pair": 1e3 * t_eq8,
                           "cores": len(os.sched_getaffinity(0)), "kind": "oracle", "cpu_model": cpu_model(),
                           "sample": f"pair 0: O6 ttcp_dense x{reps}, numpy tensordot x{reps2} (fp64)"}
        cases.append(case)
        del w, dense, Xt, Yt
        torch.cuda.empty_cache()
    clk = clocks.stop()
    line = {"mode": "example2", "metric": "Example 2 (Fig. 4a): ms per pair, TTCP incl. TT-SVD vs Eq. 8",
            "unit": "ms/pair", "higher_is_better": False, "n_gpus": 1, "dtype": "f32 (TT-SVD in f64)",
            "data": "synthetic N(0,1) dense tensors, seeded", "cases": cases, "clocks": clk}
    print(json.dumps(line))


def spawn(args):
    """--gpus N without a torch.distributed environment: re-launch this script with N ranks (one per GPU)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend, device_id=torch.device("cuda", local) if backend == "nccl" else None)
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    import paper_2109_00626_b200 as ttc
    from paper_2109_00626_b200 import dist as tdist

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = args.config
    c = ttgen.CONFIGS[cfg]
    B = args.pairs or c["B"]
    stream = torch.cuda.current_stream(dev)
    peaks, peak_kind = load_peaks()
    flush_buf = torch.empty(int(2 * L2_BYTES // 4), dtype=torch.float32, device=dev)
    if args.example2:
        if rank == 0:
            run_example2(ttc, args, dev, stream, peaks, peak_kind, flush_buf)
        return

    # ---- main line: weak scaling, this rank's B pairs (pairs rank*B .. rank*B + B - 1 of the global batch)
    w = make_work(ttc, cfg, rank * B, B, args.seed, dev, stream)
    bounds = np.arange(world + 1, dtype=np.int64) * B
    if world > 1 and c["op"] == "inner":
        def fn():
            w.step()
            tdist.gather_results(w.out, bounds)
        timed = "kernel + NCCL all_gather of the per-pair results"
    else:
        fn = w.step
        timed = "kernel" if world == 1 else "kernel (outputs stay sharded)"
    flush = w.working_set < 2 * L2_BYTES
    clocks = ClockSampler(local).start()
    time.sleep(0.3)
    t_wall0 = time.perf_counter()
    per_step_ms = time_region(fn, stream, dev, args.steps, args.warmup, flush_buf if flush else None, world)
    t_wall = time.perf_counter() - t_wall0
    clk = clocks.stop()
    ms = float(sum(per_step_ms) / len(per_step_ms))
    ms_max = max_over_ranks(ms, dev, world)
    value = B * world / (ms_max / 1e3)
    # the kernel alone (no gather) for the roofline of the dominant kernel on this rank
    if world > 1:
        k_ms = statistics.median(time_region(w.step, stream, dev, args.steps, 2, flush_buf if flush else None, world))
    else:
        k_ms = ms

    # ---- e2e: the same metric through the public API from pinned host buffers (H2D + compute + D2H)
    e2e = None
    if not args.no_e2e:
        hx = w.xin.to("cpu").pin_memory()
        hy = w.yin.to("cpu").pin_memory()
        hout = torch.empty(w.out.numel(), dtype=torch.float32).pin_memory()
        e_steps = max(3, min(args.steps, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for it in range(e_steps + 2):
            if it == 2:
                torch.cuda.synchronize(dev)
                e0.record(stream)
            w.xin.copy_(hx, non_blocking=True)
            w.yin.copy_(hy, non_blocking=True)
            w.step()
            hout.copy_(w.out, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = max_over_ranks(e0.elapsed_time(e1) / e_steps, dev, world)
        e2e = {"value": B * world / (e_ms / 1e3), "unit": UNIT, "h2d_bytes_per_step": int(4 * (hx.numel() + hy.numel())),
               "d2h_bytes_per_step": int(4 * hout.numel()), "ms_per_step": e_ms,
               "note": "per rank: pinned host -> HBM copies of the step's cores, compute, result -> host"}
        del hx, hy, hout

    roofline = roofline_for(w, k_ms, peaks, peak_kind, cfg, B)

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu:
        if hasattr(w.X, "cores"):
            Xh = ttgen.TTBatch(w.X.cores.cpu(), w.X.ranks, w.X.offsets, w.X.dims)
            Yh = ttgen.TTBatch(w.Y.cores.cpu(), w.Y.ranks, w.Y.offsets, w.Y.dims)
        else:
            Xh, Yh = w.X.cpu(), w.Y.cpu()
        cb, _, _ = cpu_oracle_rate(cfg, Xh, Yh, args.cpu_seconds, one_thread_s=3.0)
    launches = args.steps * w.launches
    w_set = w.working_set
    del w
    torch.cuda.empty_cache()

    sub = {}
    if not args.no_sub and cfg == "C2":
        for sc in [s for s in args.sub.split(",") if s]:
            sub[sc] = run_sub(ttc, sc, args, rank, world, dev, stream, peaks, peak_kind, flush_buf)

    if rank == 0:
        conf = config_dict(cfg, B, world, args.seed)
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "ours", "config": conf,
                "roofline": roofline, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": launches,
                "clocks": clk, "wall_s_timed_region": t_wall, "timed": timed,
                "l2": ("flushed between steps (2x L2 write)" if flush else
                       f"inputs ({w_set / 1e6:.0f} MB) larger than L2 ({L2_BYTES / 1e6:.0f} MB)"),
                "per_step_ms": {"min": min(per_step_ms), "median": statistics.median(per_step_ms),
                                "max": max(per_step_ms)}}
        if sub:
            line["sub"] = sub
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
