#!/usr/bin/env python
"""Benchmark of the batched TT contraction hot path (BASELINE.json metric: TT-pair contractions/s and the
fraction of the HBM/FP32 roofline).  One JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--config C2|C1|C3|C4|C5] [--impl ours|reference]

A step is one ttc_inner (or ttc_contract for C3) call over the rank's whole batch of synthetic pairs with
inputs resident in HBM.  N=1 default workload: BASELINE.json configs[1] (C2: 4096 pairs, N=8, I=16, R=16).
Multi-GPU (torchrun, one process per GPU, NCCL): every rank runs its own pairs (weak scaling: per-GPU batch
fixed), no data-path collective; device time is the max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
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


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=20)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--config", default="C2", choices=sorted(ttgen.CONFIGS))
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--pairs", type=int, default=None, help="pairs per rank (default: the config's per-GPU batch)")
    p.add_argument("--seed", type=int, default=ttgen.DEFAULT_SEED)
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU time of the oracle sample")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    return p.parse_args()


# floats of one pair's output train (uniform-rank contraction workloads): C3 ladder,
# S1 splice (chain X6^T .. X2^T, K Y2, Y3 .. Y6 of rank 8, I = 8)
PAIR_OUT = {"C3": 102976, "S1": 4224}


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
        n_el = c["I"] ** c["N"]
        shape = (c["I"],) * c["N"]
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


def per_rank_pairs(cfg: str) -> int:
    c = ttgen.CONFIGS[cfg]
    # C4 / C5 are quoted "sharded over ... 8 GPUs": one GPU's share of the 8-way split is the per-GPU batch
    return c["B"] // 8 if cfg in ("C4", "C5") else c["B"]


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


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


def flop_peak_tflops(sm_max_mhz: float) -> float:
    """FP32 FFMA peak = SMs x 128 lanes x 2 flop x max SM clock (B200_PROFILING.md unit counts)."""
    sms = torch.cuda.get_device_properties(0).multi_processor_count if torch.cuda.is_available() else 148
    return sms * 128 * 2 * sm_max_mhz * 1e6 / 1e12


# ------------------------------------------------------------------------------------------------ CPU legs
def cpu_oracle_rate(cfg: str, X, Y, target_s: float):
    """Time the oracle (as it stands) on a bounded prefix of this rank's pairs, all host cores."""
    nthreads = len(os.sched_getaffinity(0))

    def run(count):
        t0 = time.perf_counter()
        _oracle_pairs(cfg, X, Y, count, nthreads)
        return time.perf_counter() - t0

    nb = X.B if hasattr(X, "B") else X.numel() // (ttgen.CONFIGS[cfg]["I"] ** ttgen.CONFIGS[cfg]["N"])
    probe = max(1, min(nb, nthreads))
    t = run(probe)
    count = int(min(nb, max(probe, probe * target_s / max(t, 1e-6))))
    # whole passes over the sample until about target_s of CPU work (the batch may take well under target_s)
    reps, t = 0, 0.0
    while reps == 0 or (t < target_s and reps < 1000):
        t += run(count)
        reps += 1
    return {"value": reps * count / t, "unit": UNIT, "cores": nthreads, "kind": "oracle",
            "sample": f"{reps} pass(es) over the first {count} of the rank's {nb} {cfg} pairs (fp64 oracle "
                      f"{_oracle_name(cfg)}, OpenMP over pairs), {t:.1f} s"}, count, t / reps


def run_reference(args, rank, world):
    """--impl reference: the oracle timed as the reference arm (rank 0 only)."""
    if rank != 0:
        return
    cfg = args.config
    B = args.pairs or per_rank_pairs(cfg)
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
            "config": {"workload": cfg, **{k: v for k, v in ttgen.CONFIGS[cfg].items() if k != "op"},
                       "pairs_per_rank": B, "sample_pairs": count},
            "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------------ GPU arm
def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend)
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    import paper_2109_00626_b200 as ttc

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = args.config
    c = ttgen.CONFIGS[cfg]
    B = args.pairs or per_rank_pairs(cfg)
    b0 = rank * B
    if c["op"] == "alg2":
        X, Y = ttgen.dense_pairs(cfg, b0, B, args.seed, dev)
        XD = YD = None
    else:
        X, Y = ttgen.config_batch(cfg, "iid", b0, B, args.seed, dev)
        XD, YD = ttc.TTDevice.from_batch(X), ttc.TTDevice.from_batch(Y)
    stream = torch.cuda.current_stream(dev)
    launches_per_step = 1   # kernels of ours per step (counted per op below where it differs)

    if cfg == "C3":
        plan = ttc.ttc_contract_plan_create(XD, YD, c["x_modes"], c["y_modes"])
        out = torch.empty(plan.total, dtype=torch.float32, device=dev)
        in_bytes = 4.0 * (X.cores.numel() + Y.cores.numel())
        alg_bytes = in_bytes + 4.0 * plan.total
        alg_flops = 2.0 * B * 339968  # structure-aware MACs per pair

        def step():
            ttc.ttc_contract(plan, XD, YD, out=out, stream=stream)
        kernel_name = "contract_kernel"
    elif c["op"] == "splice":
        plan = ttc.ttc_splice_plan_create(XD, YD, c["x_mode"], c["y_mode"])
        out = torch.empty(plan.total, dtype=torch.float32, device=dev)
        alg_bytes = 4.0 * (X.cores.numel() + Y.cores.numel()) + 4.0 * plan.total
        # K = A_x^T A_y (I R_1 P_1 MACs) and its absorption into Y_2 (R_1 P_1 J_2 P_2 MACs), per pair
        alg_flops = 2.0 * B * (c["I"] * c["R"] * c["P"] + c["R"] * c["P"] * c["I"] * c["P"])

        def step():
            ttc.ttc_contract(plan, XD, YD, out=out, stream=stream)
        kernel_name = "splice_kernel"
    elif c["op"] == "alg2":
        # Alg. 2 on dense operands: TT-SVD of X^rho and Y^rho (step 1's permutation folded into the read),
        # K and the splice (steps 4-5), dense reconstruction in Eq. 8 order (steps 5-6)
        shape = (c["I"],) * c["N"]
        px = [c["x_mode"]] + [k for k in range(1, c["N"] + 1) if k != c["x_mode"]]
        py = [c["y_mode"]] + [k for k in range(1, c["N"] + 1) if k != c["y_mode"]]
        TX = ttc.ttc_tt_svd(X, shape, c["eps"], perm=px)
        TY = ttc.ttc_tt_svd(Y, shape, c["eps"], perm=py)
        plan = ttc.ttc_splice_plan_create(TX, TY, 1, 1)
        rx_dev = torch.from_numpy(TX.rank_rows()).to(dev)
        ry_dev = torch.from_numpy(TY.rank_rows()).to(dev)
        zc = torch.empty(plan.total, dtype=torch.float32, device=dev)
        ZD = ttc.TTDevice(zc, plan.dims, ranks=plan.ranks, offsets=plan.offsets)
        n_out = int(np.prod(plan.dims.astype(np.int64)))
        out = torch.empty(B * n_out, dtype=torch.float32, device=dev)
        rk_x = torch.empty_like(rx_dev)
        rk_y = torch.empty_like(ry_dev)
        ws_x = torch.empty(max(16, ttc.ttc_tt_svd_workspace(B, shape, px)), dtype=torch.uint8, device=dev)
        ws_y = torch.empty(max(16, ttc.ttc_tt_svd_workspace(B, shape, py)), dtype=torch.uint8, device=dev)
        n_in = c["I"] ** c["N"]
        train_x = int(sum(int(a) * int(i) * int(b2) for a, i, b2 in
                          zip(TX.rank_rows()[0][:-1], TX.dims_np, TX.rank_rows()[0][1:])))
        alg_bytes = 4.0 * B * (2 * n_in + 2 * 2 * train_x + 2 * (plan.total // B) + n_out)
        R1, I = int(TX.rank_rows()[0][1]), c["I"]
        svd_mac = 2 * (I * I * n_in // I + 2 * I ** 3 * R1 + 12 * (I - 1) * (I // 2) * I * 6)
        alg_flops = 2.0 * B * (svd_mac + I * R1 * R1 + R1 * R1 * I * R1 + n_out * R1 + 2 * I * I * R1 * R1)

        def step():
            ttc.ttc_tt_svd_into(X, shape, c["eps"], TX.cores, rk_x, perm=px, stream=stream, workspace=ws_x)
            ttc.ttc_tt_svd_into(Y, shape, c["eps"], TY.cores, rk_y, perm=py, stream=stream, workspace=ws_y)
            ttc.ttc_contract(plan, TX, TY, out=zc, stream=stream)
            ttc.ttc_reconstruct(ZD, plan.perm, out=out, stream=stream)
        kernel_name = "alg2 pipeline (ttsvd x2, splice, reconstruct)"
        # launches per step: ttc_tt_svd is 1 + 2 (N - 1) launches when every Gram side is <= 32 (the warp-Jacobi
        # pipeline, ttsvd.cu) else 1 fused launch; then the splice and the reconstruction
        dims_full = [c["I"]] * c["N"]
        side = 0
        for n in range(c["N"] - 1):
            left = int(np.prod(dims_full[:n + 1]))
            right = int(np.prod(dims_full[n + 1:]))
            side = max(side, min(left, right))
        per_svd = 1 + 2 * (c["N"] - 1) if side <= 32 else 1
        launches_per_step = 2 * per_svd + 2
    elif c["op"] == "reconstruct":
        n_el = c["I"] ** c["N"]
        out = torch.empty(B * n_el, dtype=torch.float32, device=dev)
        alg_bytes = 4.0 * X.cores.numel() + 4.0 * out.numel()
        # left / right partial products (modes 1..N/2, N/2+1..N) and their product, uniform ranks
        h = c["N"] // 2
        build = sum(c["I"] ** j * c["R"] * c["R"] for j in range(2, h + 1)) * 2
        alg_flops = 2.0 * B * (build + n_el * c["R"])

        def step():
            ttc.ttc_reconstruct(XD, None, out=out, stream=stream)
        kernel_name = "reconstruct_kernel"
    else:
        out = torch.empty(B, dtype=torch.float32, device=dev)
        mac, byts = ttc.ttc_pair_cost(XD, YD)
        alg_bytes = float(byts.sum())
        alg_flops = 2.0 * float(mac.sum())

        # heterogeneous pair costs (C5's random ranks): a cost-descending work list, computed once per batch like a
        # plan (host sort of ttc_pair_cost), so the most expensive pairs start first and the tail is short
        order = ttc.ttc_cost_order(XD, YD) if len(set(np.round(mac, 3))) > 1 else None

        def step():
            ttc.ttc_inner(XD, YD, out=out, stream=stream, order=order)
        kernel_name = "inner"

    xin = X.cores if hasattr(X, "cores") else X    # the step's device inputs (cores, or dense tensors for alg2)
    yin = Y.cores if hasattr(Y, "cores") else Y
    working_set = 4.0 * (xin.numel() + yin.numel()) + 4.0 * out.numel()
    flush = working_set < 2 * L2_BYTES
    flush_buf = torch.empty(int(2 * L2_BYTES // 4), dtype=torch.float32, device=dev) if flush else None

    for _ in range(args.warmup):
        if flush:
            flush_buf.fill_(1.0)
        step()
    torch.cuda.synchronize(dev)

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    clocks = ClockSampler(local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize(dev)
    clocks.start()
    time.sleep(0.3)
    t_wall0 = time.perf_counter()
    for k in range(args.steps):
        if flush:
            flush_buf.fill_(float(k))
        starts[k].record(stream)
        step()
        ends[k].record(stream)
    torch.cuda.synchronize(dev)
    t_wall = time.perf_counter() - t_wall0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    per_step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = float(sum(per_step_ms) / len(per_step_ms))
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = B * world / (ms_max / 1e3)

    # ---- e2e: the same metric through the public API from pinned host buffers (H2D + compute + D2H)
    e2e = None
    if not args.no_e2e:
        hx = xin.to("cpu").pin_memory()
        hy = yin.to("cpu").pin_memory()
        hout = torch.empty(out.numel(), dtype=torch.float32).pin_memory()
        e_steps = max(3, min(args.steps, 10))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for it in range(e_steps + 2):
            if it == 2:
                torch.cuda.synchronize(dev)
                e0.record(stream)
            xin.copy_(hx, non_blocking=True)
            yin.copy_(hy, non_blocking=True)
            step()
            hout.copy_(out, non_blocking=True)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        e_ms = e0.elapsed_time(e1) / e_steps
        et = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": B * world / (float(et.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(4 * (hx.numel() + hy.numel())), "d2h_bytes_per_step": int(4 * hout.numel()),
               "ms_per_step": float(et.item())}

    peaks, peak_kind = load_peaks()
    achieved_gbs = alg_bytes / (ms / 1e3) / 1e9
    fp32_peak = flop_peak_tflops(float(peaks.get("sm_max_mhz", 1965.0)))
    achieved_tf = alg_flops / (ms / 1e3) / 1e12
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(cfg)
        except Exception:
            traffic = None
    hbm = {"bound": "hbm", "achieved": achieved_gbs, "peak": float(peaks["hbm_gbs"]), "unit": "GB/s",
           "frac": achieved_gbs / float(peaks["hbm_gbs"]), "traffic": traffic,
           "peak_source": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs: copy bandwidth)",
           "algorithmic_bytes_per_launch": alg_bytes}
    # FP32 arithmetic roofline (north star: "the slower of the sweep's FLOPs at FP32 peak and the core bytes at
    # HBM bandwidth"); the peak is derived from unit counts and clocks, hence "alu".
    alu = {"bound": "alu", "achieved": achieved_tf, "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved_tf / fp32_peak,
           "traffic": traffic, "peak_source": "148 SMs x 128 FP32 lanes x 2 flop x sm_max_mhz (B200_PROFILING.md unit counts)",
           "algorithmic_flops_per_launch": alg_flops}
    t_hbm = alg_bytes / (peaks["hbm_gbs"] * 1e9)
    t_alu = alg_flops / (fp32_peak * 1e12)
    top, other = (hbm, alu) if t_hbm >= t_alu else (alu, hbm)
    roofline = dict(top)
    roofline.update({"kernel": kernel_name, "other": {k: v for k, v in other.items() if k != "traffic"},
                     "frac_vs_spec_8TBs": achieved_gbs / 8000.0})

    cb = None
    if rank == 0 and world == 1 and not args.no_cpu:
        if hasattr(X, "cores"):
            Xh = ttgen.TTBatch(X.cores.cpu(), X.ranks, X.offsets, X.dims)
            Yh = ttgen.TTBatch(Y.cores.cpu(), Y.ranks, Y.offsets, Y.dims)
        else:
            Xh, Yh = X.cpu(), Y.cpu()
        cb, _, _ = cpu_oracle_rate(cfg, Xh, Yh, args.cpu_seconds)

    if rank == 0:
        conf = {"workload": cfg, **{k: (list(v) if isinstance(v, tuple) else v) for k, v in c.items() if k != "op"},
                "op": c["op"], "pairs_per_rank": B, "global_pairs": B * world, "seed": args.seed,
                "l2": ("flushed between steps (2x L2 write)" if flush else
                       f"inputs ({working_set / 1e6:.0f} MB) larger than L2 ({L2_BYTES / 1e6:.0f} MB)"),
                "parallelism": f"dp{world}"}
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "ours", "config": conf,
                "roofline": roofline, "cpu_baseline": cb, "e2e": e2e, "gpu_launches": args.steps * launches_per_step,
                "clocks": clk, "wall_s_timed_region": t_wall,
                "per_step_ms": {"min": min(per_step_ms), "median": statistics.median(per_step_ms),
                                "max": max(per_step_ms)}}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
