#!/usr/bin/env python
"""Benchmark of the CPO/CPS sparse-conv hot path on B200 (contract: see DESIGN.md §Measurement).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg2]

One step = one pass of the hot path over one batch of the workload: CPO encode
(one launch) + sparse convolution (one launch) of configs[1] (cfg2: 1x64x56x56,
rho 0.3, 64 output channels, 3x3, s1, pad 1).  Inputs are synthetic (seeded
clustered-ReLU, DESIGN.md §Input recipe) and resident in HBM; L2 is flushed
between timed steps.  value = dense-equivalent GFLOP/s (2*N*K*C*R*S*Oh*Ow per
step / device time), summed over ranks (weak scaling: every rank encodes and
convolves its own batch; no data-path collective).  The same line carries the
CPS path, the im2col baseline (lowering + GEMM), the compression ratio, the
roofline of the dominant kernel, the host-buffer end-to-end number, clocks and
the oracle timed on the host (cpu_baseline).

--impl reference runs the CPU oracle (oracle/, plain C, FP64) as the reference
arm on the same workload, on the host, rank 0 only.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from synth import CATALOG, CONFIGS, cfg5_layers, clustered_relu, he_normal  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
SM_COUNT, FP32_LANES, FALLBACK_HBM = 148, 128, 6650.0
METRIC = "dense-equivalent GFLOP/s of CPO encode + sparse conv (per layer), vs GPU im2col"


def workload(name: str):
    if name.startswith("cfg5"):
        layer = cfg5_layers(batch=32)[int(name.split("L")[-1])]
        return layer
    if name in CATALOG:
        return CATALOG[name]
    return CONFIGS[name]


def dense_flops(d, Oh, Ow):
    return 2.0 * d["N"] * d["K"] * d["C"] * d["R"] * d["S"] * Oh * Ow


def nze_macs(d, x: np.ndarray, Oh, Ow) -> int:
    """Exact multiply-adds of the sparse conv: for each NZE, the (output, tap) pairs
    that see it (rows x cols, stride-aware), times K.  Measurement accounting only."""
    Hp, Wp = d["H"] + d["pad_top"] + d["pad_bottom"], d["W"] + d["pad_left"] + d["pad_right"]

    def cov(n_in, k, s, n_out):
        c = np.zeros(n_in, dtype=np.int64)
        for h in range(n_in):
            c[h] = sum(1 for l in range(k) if h - l >= 0 and (h - l) % s == 0 and (h - l) // s < n_out)
        return c
    ch = cov(Hp, d["R"], d["stride_h"], Oh)[d["pad_top"]:d["pad_top"] + d["H"]]
    cw = cov(Wp, d["S"], d["stride_w"], Ow)[d["pad_left"]:d["pad_left"] + d["W"]]
    nz = (x != 0).sum(axis=(0, 1)).astype(np.int64)      # [H, W]
    return int(ch @ nz @ cw) * d["K"]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def tf32_peak():
    """Dense TF32 tensor peak, TFLOP/s: the measured bf16 peak (MEASURED_PEAKS.json) times the
    guide's nominal tf32 / bf16 ratio (1.1 / 2.25 PFLOP/s, B200_PROFILING.md)."""
    try:
        with open(PEAKS_FILE) as f:
            return float(json.load(f)["bf16_tflops"]) * 1.1 / 2.25
    except Exception:
        return 1100.0


def load_peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p.get("sm_max_mhz", 1965.0)), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return FALLBACK_HBM, 1965.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clock + throttle reasons sampled with NVML every ~1 ms during the timed region."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index: int):
        self.index, self.rows, self.stop = index, [], threading.Event()

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.maxclk = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self._sample()
            self.t = threading.Thread(target=self._loop, daemon=True)
            self.t.start()
        except Exception:
            self.nv = None
        return self

    def _sample(self):
        clk = self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM)
        rs = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.rows.append((clk, rs))

    def _loop(self):
        while not self.stop.is_set():
            try:
                self._sample()
            except Exception:
                break
            time.sleep(0.001)

    def __exit__(self, *a):
        self.stop.set()
        if self.nv is not None:
            self.t.join(timeout=1)
            try:
                self._sample()
            except Exception:
                pass

    def summary(self):
        if not self.rows or self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        reasons = sorted({n for _, r in self.rows for n, bit in self.REASONS.items() if r & bit})
        return {"sm_mhz": statistics.median(c for c, _ in self.rows), "sm_max_mhz": self.maxclk,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------- CPU oracle legs

def oracle_time(d, x, w, budget_s: float, cps: bool = False):
    """Oracle encode + sparse conv (Alg. 1/2 or 3/4, single-threaded C) on a bounded
    sample: as many images of the batch as fit the budget (at least one)."""
    import oracle
    oracle.build()
    t_used, n_done, flops = 0.0, 0, 0.0
    Oh, Ow = oracle.out_hw(d)
    d1 = dict(d, N=1)
    while n_done < d["N"] and (n_done == 0 or t_used < budget_s):
        xi = x[n_done:n_done + 1]
        t0 = time.perf_counter()
        enc = oracle.encode(d1, xi, cps=cps)
        oracle.sparse_conv(d1, enc, w)
        t_used += time.perf_counter() - t0
        flops += dense_flops(d1, Oh, Ow)
        n_done += 1
    return t_used, n_done, flops


def oracle_time_threads(d, x, w, budget_s: float, threads: int):
    """The same oracle calls on all host cores: per image, the CPO encode (one thread),
    then Alg. 2 over disjoint output-channel slices in parallel threads (the C oracle is
    reentrant and ctypes releases the GIL).  The oracle itself is unchanged."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    oracle.build()
    Oh, Ow = oracle.out_hw(d)
    d1 = dict(d, N=1)
    K = d["K"]
    bounds = [(K * i // threads, K * (i + 1) // threads) for i in range(threads)]
    bounds = [(a, b) for a, b in bounds if b > a]
    t_used, n_done, flops = 0.0, 0, 0.0
    with ThreadPoolExecutor(len(bounds)) as ex:
        while n_done < d["N"] and (n_done == 0 or t_used < budget_s):
            xi = x[n_done:n_done + 1]
            t0 = time.perf_counter()
            enc = oracle.encode(d1, xi)
            list(ex.map(lambda ab: oracle.sparse_conv(dict(d1, K=ab[1] - ab[0]), enc, w[ab[0]:ab[1]]), bounds))
            t_used += time.perf_counter() - t0
            flops += dense_flops(d1, Oh, Ow)
            n_done += 1
    return t_used, n_done, flops, len(bounds)


def oracle_legs(d, x, w):
    """The oracle's other algorithms on one image, single thread: CPS encode +
    Alg. 4, the direct nested-loop conv (Eq. 1) and im2col + naive GEMM; dense-equiv. GFLOP/s."""
    import oracle
    oracle.build()
    d1 = dict(d, N=1)
    Oh, Ow = oracle.out_hw(d1)
    f = dense_flops(d1, Oh, Ow)
    xi = x[:1]
    out = {}
    for name, fn in (("cps", lambda: oracle.sparse_conv(d1, oracle.encode(d1, xi, cps=True), w)),
                     ("direct", lambda: oracle.direct_conv(d1, xi, w)),
                     ("im2col_gemm", lambda: oracle.gemm_lowered(d1, oracle.im2col(d1, xi), w))):
        t0 = time.perf_counter()
        fn()
        out[name] = f / (time.perf_counter() - t0) / 1e9
    out["unit"] = "GFLOP/s (dense-equivalent, one image, one thread)"
    return out


def run_reference(args):
    """--impl reference: the oracle as the reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    c = workload(args.workload)
    d = c["desc"]
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], c["seed"], c["dead_frac"], c["zero_tile_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    for _ in range(args.warmup):
        oracle_time(d, x[:1], w, 0.0)
    tot_t, tot_f, imgs = 0.0, 0.0, 0
    for _ in range(args.steps):
        t, n, f = oracle_time(d, x, w, budget_s=20.0 / max(1, args.steps))
        tot_t, tot_f, imgs = tot_t + t, tot_f + f, imgs + n
    val = tot_f / tot_t / 1e9
    line = {"impl": "reference", "metric": METRIC,
            "value": val, "unit": "GFLOP/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.workload, **{k: d[k] for k in d}, "density": c["density"]},
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
                             "sample": f"{imgs} image(s) of {args.workload} over {args.steps} steps"},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------- cfg5 stack leg

def run_stack(args, world, rank, dev, flush, hbm_gbs, p_fp32):
    """cfg5: global batch args.stack_batch sharded over the ranks (strong scaling of this
    sub-metric), per-layer plan selected offline on rank 0 and broadcast, the 16 layers
    captured in one CUDA graph, then the one output gather (NCCL all-gather).
    images/s = global batch / max over ranks of (stack + gather) device time."""
    import torch
    import torch.distributed as dist

    import paper_2104_08314_b200 as spc
    from paper_2104_08314_b200.stack import Cfg5Stack, broadcast_plan, gather_outputs, shard_range
    lo, hi = shard_range(args.stack_batch, world, rank)
    S = Cfg5Stack(hi - lo, dev, rank=rank)
    plan = S.select(args.stack_mode) if rank == 0 else None
    plan = broadcast_plan(plan)
    S.set_plan(plan)
    graph = S.capture()
    stream = torch.cuda.current_stream()
    n_per_rank = [shard_range(args.stack_batch, world, r)[1] - shard_range(args.stack_batch, world, r)[0]
                  for r in range(world)]
    for _ in range(3):
        graph.replay()
        gather_outputs(S.layers[-1].y, n_per_rank)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.stack_steps)]
    for i in range(args.stack_steps):
        flush.zero_()
        ev[i][0].record(stream)
        graph.replay()
        ev[i][1].record(stream)
        out = gather_outputs(S.layers[-1].y, n_per_rank)
        ev[i][2].record(stream)
    torch.cuda.synchronize()
    t_stack = sum(a.elapsed_time(b) for a, b, _ in ev) / args.stack_steps
    t_gather = sum(b.elapsed_time(c) for _, b, c in ev) / args.stack_steps
    tt = torch.tensor([t_stack, t_gather, t_stack + t_gather], device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    t_stack, t_gather, t_tot = (float(v) for v in tt.tolist())
    assert out.shape[0] == args.stack_batch
    # roofline of the chosen plan (per-layer t_roof = max(bytes / HBM, FLOPs / peak of its engine))
    t_roof = 0.0
    layers = []
    for sp, L, algo, xb in zip(S.specs, S.layers, S.plan, S.host_inputs):
        d = sp["desc"]
        Oh, Ow = L.Oh, L.Ow
        reps = (d["N"] + xb.shape[0] - 1) // xb.shape[0]
        x_bytes = 4 * d["N"] * d["C"] * d["H"] * d["W"]
        y_bytes = 4 * d["N"] * d["K"] * Oh * Ow
        w_bytes = 4 * d["K"] * d["C"] * d["R"] * d["S"]
        if algo == "im2col":
            low = 4 * d["N"] * d["C"] * d["R"] * d["S"] * Oh * Ow
            if spc.spc_im2col_engine(d) == spc.SPC_GEMM_TC_3XTF32:
                # three TF32 products per fp32 MAC at the TF32 tensor peak
                t_mma = 3 * dense_flops(d, Oh, Ow) / (tf32_peak() * 1e12)
            else:
                t_mma = dense_flops(d, Oh, Ow) / (p_fp32 * 1e12)
            tr = max((x_bytes + 2 * low + w_bytes + y_bytes) / (hbm_gbs * 1e9), t_mma)
        else:
            macs = nze_macs(dict(d, N=xb.shape[0]), xb, Oh, Ow) * reps * (d["N"] / (xb.shape[0] * reps))
            nnz = int((xb != 0).sum()) * d["N"] / xb.shape[0]
            enc_bytes = x_bytes + 8 * nnz + 8 * 3 * d["N"] * d["C"]
            tr = max(enc_bytes / (hbm_gbs * 1e9), 0) + max((8 * nnz + w_bytes + y_bytes) / (hbm_gbs * 1e9),
                                                          2.0 * macs / (p_fp32 * 1e12))
        t_roof += tr
        layers.append({"layer": sp["name"], "density": round(sp["density"], 4), "algo": algo})
    res = {"workload": "cfg5 ResNet-50 3x3 stack (16 layers)", "global_batch": args.stack_batch,
           "per_rank_batch": hi - lo, "n_gpus": world, "mode": args.stack_mode,
           "images_per_s": args.stack_batch / (t_tot * 1e-3), "ms_per_step": t_tot, "stack_ms": t_stack,
           "gather_ms": t_gather, "gather": "NCCL all_gather_into_tensor of the last layer's output" if world > 1
           else "none (1 GPU)", "steps": args.stack_steps, "scaling": "strong (global batch fixed)",
           "roofline_images_per_s": (hi - lo) / t_roof if t_roof > 0 else None,
           "roofline_frac": (t_roof * 1e3) / t_tot if t_tot > 0 else None,
           "roofline_model": "sum over layers of the chosen algorithm's bound: sparse = encode bytes / HBM + "
                             "max(compressed + weight + output bytes / HBM, NZE FLOPs / FP32 peak); im2col = "
                             "max(x + 2 x lowered + w + y bytes / HBM, dense FLOPs / FP32 peak (cuBLAS FP32) or "
                             "3 x dense FLOPs / TF32 tensor peak (tcgen05 3xTF32))",
           "plan": layers, "select_ms_per_sample": S.select_times if rank == 0 else None,
           "gemm": spc.GEMM_NAMES[spc.spc_get_im2col_gemm()],
           "gemm_per_layer": [spc.GEMM_NAMES[spc.spc_im2col_engine(sp["desc"])] for sp in S.specs],
           "inputs": "8 distinct seeded clustered-ReLU images per layer, tiled to the batch; L2 flushed per step"}
    if rank == 0 and not args.no_cpu:
        import oracle
        oracle.build()
        t_cpu = 0.0
        for sp, xb, w in zip(S.specs, S.host_inputs, S.weights):
            t, n, _ = oracle_time(dict(sp["desc"], N=2), xb[:2], w, budget_s=1e9)
            t_cpu += t
        res["cpu_baseline"] = {"value": 2 / t_cpu, "unit": "images/s", "cores": 1, "kind": "oracle",
                               "sample": "2 images through all 16 layers: oracle CPO encode + Alg. 2 conv, "
                                         "single thread, FP64"}
    return res


# ---------------------------------------------------------------- GPU leg

def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2104_08314_b200 as spc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream()

    c = workload(args.workload)
    d = c["desc"]
    # each rank draws its own images (weak scaling: independent batches)
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], c["seed"] + 7919 * rank, c["dead_frac"],
                       c["zero_tile_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    from paper_2104_08314_b200.layer import SparseConvLayer
    Oh, Ow = spc.out_hw(d)
    xg = torch.from_numpy(x).to(dev)
    wg = torch.from_numpy(w).to(dev)
    L_cpo = SparseConvLayer(d, wg, device=dev)
    L_cps = SparseConvLayer(d, wg, device=dev)
    y = L_cpo.y
    enc, enc_s = L_cpo.enc, L_cps.enc
    flush = torch.empty(int(2 * 128 * 2 ** 20) // 4, dtype=torch.float32, device=dev)  # > 2x L2

    # CUDA graphs of each step: the host enqueues a whole step at once, so the
    # device timeline between the events holds only our kernels.
    g_cpo = L_cpo.capture(lambda: L_cpo.forward(xg, "cpo"))
    g_cpo_enc = L_cpo.capture(lambda: L_cpo.encode(xg, "cpo"))
    g_cpo_conv = L_cpo.capture(lambda: L_cpo.conv())
    g_cps = L_cps.capture(lambda: L_cps.forward(xg, "cps"))
    g_cps_enc = L_cps.capture(lambda: L_cps.encode(xg, "cps"))
    g_i2c = L_cpo.capture(lambda: L_cpo.forward(xg, "im2col"))
    L_cpo.forward(xg, "cpo")       # leave the CPO encoding in place for the conv-only graph

    step_ms = {}

    def timed(graph, steps, warmup, flush_l2=True, key=None):
        for _ in range(warmup):
            graph.replay()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for i in range(steps):
            if flush_l2:
                flush.zero_()                  # L2 flush between timed steps (outside the events)
            ev[i][0].record(stream)
            graph.replay()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        ts = [a.elapsed_time(b) for a, b in ev]
        if key:
            step_ms[key] = ts
        return sum(ts)

    # --- main timed region (CPO path), barrier + sync on both sides, max over ranks
    for _ in range(args.warmup):
        g_cpo.replay()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        t_ms = timed(g_cpo, args.steps, 0, key="cpo")
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    tmax = t_ms
    if world > 1:
        tt = torch.tensor([t_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        tmax = float(tt.item())
    flops_step = dense_flops(d, Oh, Ow)
    value = flops_step * args.steps * world / (tmax * 1e-3) / 1e9

    # --- per-kernel breakdown and the other algorithms (same process)
    t_hot_ms = timed(g_cpo, args.steps, 1, flush_l2=False)   # hot L2: no flush
    t_enc_ms = timed(g_cpo_enc, args.steps, 1)
    t_conv_ms = timed(g_cpo_conv, args.steps, 1)
    t_cps = timed(g_cps, args.steps, 1)
    t_cps_enc = timed(g_cps_enc, args.steps, 1)
    t_i2c = timed(g_i2c, args.steps, 1)

    # Per-launch kernel durations for the rooflines: timing events recorded INSIDE a
    # graph right around the one kernel (external event-record nodes on the stream
    # the kernel is launched on), an L2 flush before each, so the graph launch and
    # the event round trip to the host (~6 us per step on this pool) are not in it.
    def kernel_timed(fn, steps, reps=50):
        reps = max(1, min(reps, steps))
        evs = [(torch.cuda.Event(enable_timing=True, external=True),
                torch.cuda.Event(enable_timing=True, external=True)) for _ in range(reps)]

        def body():
            for a, b in evs:
                flush.zero_()
                a.record()
                fn()
                b.record()
        g = L_cpo.capture(body, warmup=1)
        ts = []
        for _ in range(max(1, steps // reps) + 1):   # first replay is warm-up
            g.replay()
            torch.cuda.synchronize()
            ts.append([a.elapsed_time(b) for a, b in evs])
        ts = [t for row in ts[1:] for t in row]
        return float(np.mean(ts)), float(np.median(ts))

    k_conv_ms, k_conv_med = kernel_timed(lambda: L_cpo.conv(), args.steps)
    k_enc_ms, k_enc_med = kernel_timed(lambda: L_cpo.encode(xg, "cpo"), args.steps)
    L_cpo.forward(xg, "cpo")

    # encoding sizes, CR (paper units: elements of ptr + DA + IN vs S_im2col)
    pl_, dl_, il_ = spc.spc_encoding_lengths(enc)
    ps_, ds_, is_ = spc.spc_encoding_lengths(enc_s)
    s_im2col = d["N"] * Oh * Ow * d["C"] * d["R"] * d["S"]
    side = 3 * (d["N"] * d["C"] + 1) * 2   # int64 side tables in 4-byte elements
    cr_cpo = s_im2col / (pl_ + dl_ + il_)
    cr_cps = s_im2col / (ps_ + ds_ + is_)

    # --- roofline of the dominant kernel (measured per-launch averages)
    hbm_gbs, sm_max_mhz, peak_src = load_peaks()
    p_fp32 = SM_COUNT * FP32_LANES * 2 * sm_max_mhz * 1e6 / 1e12   # TFLOP/s, derived
    macs = nze_macs(d, x, Oh, Ow)
    conv_bytes = 4 * (pl_ + dl_ + il_) + 8 * 2 * (d["N"] * d["C"] + 1) + 4 * wg.numel() + 4 * y.numel()
    enc_bytes = 4 * xg.numel() + 4 * (pl_ + dl_ + il_) + 8 * 3 * (d["N"] * d["C"] + 1)
    conv_s = k_conv_ms * 1e-3          # average launch duration (in-graph events)
    enc_s = k_enc_ms * 1e-3
    conv_flops = 2.0 * macs
    t_roof_conv = max(conv_bytes / (hbm_gbs * 1e9), conv_flops / (p_fp32 * 1e12))
    conv_bound = "alu" if conv_flops / (p_fp32 * 1e12) >= conv_bytes / (hbm_gbs * 1e9) else "hbm"
    traffic = None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            traffic = json.load(open(tfile)).get(args.workload, {}).get("sparse_conv")
        except Exception:
            traffic = None
    if conv_s >= enc_s:
        if conv_bound == "alu":
            roof = {"kernel": "strip_conv_kernel (sparse conv)", "bound": "alu", "achieved": conv_flops / conv_s / 1e12,
                    "peak": p_fp32, "unit": "TFLOP/s", "frac": t_roof_conv / conv_s, "traffic": traffic,
                    "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 x max SM clock",
                    "algorithmic_flops": conv_flops, "algorithmic_bytes": conv_bytes,
                    "duration_us": conv_s * 1e6}
        else:
            roof = {"kernel": "strip_conv_kernel (sparse conv)", "bound": "hbm", "achieved": conv_bytes / conv_s / 1e9,
                    "peak": hbm_gbs, "unit": "GB/s", "frac": t_roof_conv / conv_s, "traffic": traffic,
                    "peak_source": peak_src, "algorithmic_bytes": conv_bytes}
    else:
        roof = {"kernel": "encode_kernel", "bound": "hbm", "achieved": enc_bytes / enc_s / 1e9, "peak": hbm_gbs,
                "unit": "GB/s", "frac": enc_bytes / enc_s / 1e9 / hbm_gbs, "traffic": None,
                "peak_source": peak_src, "algorithmic_bytes": enc_bytes}

    # --- end to end through the public API with host buffers: pinned H2D of the
    # input, encode + conv, D2H of the output, all inside the timed region
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty(y.shape, dtype=torch.float32).pin_memory()

    def e2e_step():
        xg.copy_(xh, non_blocking=True)
        L_cpo.forward(xg, "cpo")
        yh.copy_(y, non_blocking=True)
    g_e2e = L_cpo.capture(e2e_step)
    e2e_serial_ms = timed(g_e2e, args.steps, 2)

    # Pipelined form of the same steps (what a serving loop does): two layer instances
    # with their own input / encoding / output buffers; per step, H2D on one stream,
    # encode + conv on a second, D2H on a third, so step i's copies overlap the
    # neighbouring steps' compute.  One graph holds PIPE steps (fill and drain included);
    # every step still copies its whole input in and its whole output out.
    PIPE = 16
    Ls = [L_cpo, SparseConvLayer(d, wg, device=dev)]
    xgs = [xg, torch.empty_like(xg)]
    yhs = [yh, torch.empty(y.shape, dtype=torch.float32).pin_memory()]
    s_h, s_c, s_d = (torch.cuda.Stream(device=dev) for _ in range(3))
    ev_h = [torch.cuda.Event() for _ in range(PIPE)]
    ev_c = [torch.cuda.Event() for _ in range(PIPE)]
    ev_d = [torch.cuda.Event() for _ in range(PIPE)]

    def pipeline():
        cs = torch.cuda.current_stream()
        for st_ in (s_h, s_c, s_d):
            st_.wait_stream(cs)
        for i in range(PIPE):
            b = i & 1
            with torch.cuda.stream(s_h):
                if i >= 2:
                    s_h.wait_event(ev_c[i - 2])      # xg[b] free: step i-2's encode read it
                xgs[b].copy_(xh, non_blocking=True)
                ev_h[i].record(s_h)
            with torch.cuda.stream(s_c):
                s_c.wait_event(ev_h[i])
                if i >= 2:
                    s_c.wait_event(ev_d[i - 2])      # y[b] free: step i-2's D2H read it
                Ls[b].forward(xgs[b], "cpo")
                ev_c[i].record(s_c)
            with torch.cuda.stream(s_d):
                s_d.wait_event(ev_c[i])
                yhs[b].copy_(Ls[b].y, non_blocking=True)
                ev_d[i].record(s_d)
        for st_ in (s_h, s_c, s_d):
            cs.wait_stream(st_)
    for _ in range(2):
        pipeline()
    torch.cuda.synchronize()
    g_pipe = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g_pipe):
        pipeline()
    reps = max(1, args.steps // PIPE)
    e2e_ms = timed(g_pipe, reps, 2) * args.steps / (reps * PIPE)   # per-step mean, scaled to K steps
    if world > 1:
        tt = torch.tensor([e2e_ms, e2e_serial_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms, e2e_serial_ms = float(tt[0].item()), float(tt[1].item())
    e2e_val = flops_step * args.steps * world / (e2e_ms * 1e-3) / 1e9

    cpu = None
    if rank == 0 and not args.no_cpu:
        t, n, f = oracle_time(d, x, w, budget_s=args.cpu_budget)
        cpu = {"value": f / t / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
               "host_cpus": os.cpu_count(), "cpu_model": cpu_model(),
               "sample": f"{n} image(s) of {args.workload}: oracle CPO encode + Alg. 2 conv, single thread, FP64"}
        cpu["legs"] = oracle_legs(d, x, w)
        t2, n2, f2, thr = oracle_time_threads(d, x, w, args.cpu_budget, os.cpu_count() or 1)
        cpu["all_cores"] = {"value": f2 / t2 / 1e9, "unit": "GFLOP/s", "cores": thr,
                            "sample": f"{n2} image(s): encode on one thread, Alg. 2 over {thr} output-channel "
                                      "slices in parallel threads"}

    stack = None
    if not args.no_stack:
        stack = run_stack(args, world, rank, dev, flush, hbm_gbs, p_fp32)

    if world > 1:
        dist.barrier()
    if rank == 0:
        us = lambda ms: 1e3 * ms / args.steps  # noqa: E731
        line = {
            "metric": METRIC,
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "ms_per_step_median": float(np.median(step_ms["cpo"])) if rank == 0 else None,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, **{k: d[k] for k in d}, "density": c["density"],
                       "dead_frac": c["dead_frac"], "zero_tile_frac": c["zero_tile_frac"],
                       "l2": "flushed between timed steps (256 MiB write)", "global_batch": d["N"] * world},
            "layer_us": {"cpo_encode": us(t_enc_ms), "cpo_conv": us(t_conv_ms), "cpo_total": us(t_ms),
                         "cpo_total_hot_l2": us(t_hot_ms),
                         "cps_encode": us(t_cps_enc), "cps_conv": us(t_cps - t_cps_enc), "cps_total": us(t_cps),
                         "im2col_total": us(t_i2c)},
            "kernel_us": {"timing": "per launch, timing events inside a graph around the one kernel, L2 flushed before each",
                          "cpo_conv_mean": 1e3 * k_conv_ms, "cpo_conv_median": 1e3 * k_conv_med,
                          "cpo_encode_mean": 1e3 * k_enc_ms, "cpo_encode_median": 1e3 * k_enc_med},
            "im2col": {"value": flops_step * args.steps / (t_i2c * 1e-3) / 1e9, "unit": "GFLOP/s",
                       "gemm": spc.GEMM_NAMES[spc.spc_im2col_engine(d)]},
            "speedup_vs_im2col": t_i2c / t_ms,
            "cr": {"cpo": cr_cpo, "cps": cr_cps, "cpo_with_side_tables": s_im2col / (pl_ + dl_ + il_ + side),
                   "ptr": pl_, "da": dl_, "in_cpo": il_, "in_cps": is_, "S_im2col": s_im2col},
            "nze_macs": macs, "density_measured": float((x != 0).mean()),
            "roofline": roof,
            "roofline_encode": {"bound": "hbm", "achieved": enc_bytes / enc_s / 1e9, "peak": hbm_gbs,
                                "unit": "GB/s", "frac": enc_bytes / enc_s / 1e9 / hbm_gbs},
            "e2e": {"value": e2e_val, "unit": "GFLOP/s", "h2d_bytes_per_step": int(4 * xg.numel()),
                    "d2h_bytes_per_step": int(4 * y.numel()), "ms_per_step": e2e_ms / args.steps,
                    "form": f"pipelined: H2D / encode+conv / D2H on three streams, {PIPE} steps per graph "
                            "(fill and drain included), two buffer sets; no L2 flush inside the graph "
                            "(each step's input arrives from the host)",
                    "serial": {"value": flops_step * args.steps * world / (e2e_serial_ms * 1e-3) / 1e9,
                               "ms_per_step": e2e_serial_ms / args.steps,
                               "form": "one step per graph: H2D, encode, conv, D2H in sequence"}},
            "gpu_launches": 2 * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "stack": stack,
            "version": spc.spc_version(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stack", action="store_true", help="skip the cfg5 stack leg")
    ap.add_argument("--stack-batch", type=int, default=256)
    ap.add_argument("--stack-steps", type=int, default=10)
    ap.add_argument("--stack-mode", default="best_of_three", choices=["favour_time", "favour_space", "best_of_three"])
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        print("warning: fewer than 3 warm-up steps", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
