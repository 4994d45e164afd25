#!/usr/bin/env python
"""Benchmark of the CPO/CPS sparse-conv hot path on B200 (contract: see DESIGN.md §8).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfg3]

One step = one pass of the hot path over one batch of the workload: CPO encode
(one launch) + sparse convolution (one launch).  The headline workload is
BASELINE.json configs[2] (cfg3: 8x256x14x14, rho 0.1, 20% dead channels,
256 output channels, 3x3, s1, pad 1), the largest single-layer configuration.
Inputs are synthetic (seeded clustered-ReLU) and resident in HBM.
L2: steps run back to back over NSET copies of the layer's buffers (input,
encoding, workspace, packed weights, output) whose bytes touched per cycle
exceed 1.5x the 126 MB L2, so every step reads its data cold ("inputs larger
than L2"); configurations too small for that (cfg1) flush L2 between steps
instead, and say so.  value = dense-equivalent GFLOP/s (2*N*K*C*R*S*Oh*Ow per
step / device time), summed over ranks (weak scaling: every rank encodes and
convolves its own batch; no data-path collective).  The same line carries
per-kernel launch durations, the roofline of the dominant kernel, per-config
rows (cfg1..cfg4, the cfg3 stride-2 layer and density sweep), the im2col
baseline, the compression ratio, the host-buffer end-to-end number, clocks,
the cfg5 stack (offline selection and forced CPO) and the oracle timed on the
host (cpu_baseline).

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
            # the same config object as the GPU arm's line (its L2 plan is host arithmetic)
            "config": {"workload": args.workload, **{k: d[k] for k in d}, "density": c["density"],
                       "dead_frac": c["dead_frac"], "zero_tile_frac": c["zero_tile_frac"],
                       "l2": l2_note_of(*l2_plan(d, make_pool(c, 0))), "global_batch": d["N"] * max(1, args.gpus)},
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
                             "sample": f"{imgs} image(s) of {args.workload} over {args.steps} steps"},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


# ---------------------------------------------------------------- rotating buffers

L2_BYTES = 126 * 2 ** 20


class Rotating:
    """NSET copies of one layer's device buffers (input, encoding, workspace, packed weights,
    output; lowered matrix for im2col) so that back-to-back steps cycle through more bytes
    than L2 holds: every step reads its data cold without an L2 flush between steps."""

    def __init__(self, d, pool: np.ndarray, w: np.ndarray, dev, min_sets=4, max_sets=128, relu=False):
        import torch
        from paper_2104_08314_b200.layer import SparseConvLayer
        self.d, self.dev = d, dev
        N = d["N"]
        self.nset, self.cold, self.touched = l2_plan(d, pool, min_sets, max_sets)
        self.layers, self.xs = [], []
        nd = pool.shape[0]
        for i in range(self.nset):
            idx = [(i + j) % nd for j in range(N)]     # rotate the distinct images through the batch
            self.xs.append(torch.from_numpy(np.ascontiguousarray(pool[idx])).to(dev))
            self.layers.append(SparseConvLayer(d, torch.from_numpy(w).to(dev), device=dev, relu=relu))
        self.flush = None if self.cold else torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device=dev)
        self._graphs = {}

    def graph(self, kind: str, n: int):
        """One CUDA graph of n consecutive steps of `kind` (sets 0..n-1): step / encode / conv /
        cps / im2col.  The host enqueues n steps at once; inside the graph the kernels run
        back to back (PDL overlaps a conv's prologue with its encoder)."""
        import torch
        key = (kind, n)
        if key in self._graphs:
            return self._graphs[key]
        Ls, xs = self.layers, self.xs

        def body():
            for i in range(n):
                L, x = Ls[i % self.nset], xs[i % self.nset]
                if kind == "step":
                    L.forward(x, "cpo")
                elif kind == "encode":
                    L.encode(x, "cpo")
                elif kind == "conv":
                    L.conv()
                elif kind == "cps":
                    L.forward(x, "cps")
                elif kind in ("im2col", "cscc", "cpo_sa"):
                    L.forward(x, kind)
        # warm the buffers (lowered workspaces, the encodings the conv-only graph reads)
        body()
        torch.cuda.synchronize()
        g = Ls[0].capture(body, warmup=1)
        self._graphs[key] = g
        return g

    def timed(self, kind: str, steps: int, stream) -> float:
        """Device ms of exactly `steps` steps of `kind`: back to back over the rotating sets
        (full cycles as one graph, the remainder as a second), or -- for a configuration too
        small to exceed L2 -- one step per replay with a 2x-L2 write between steps."""
        import torch
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        if not self.cold:
            g = self.graph(kind, 1)
            tot = 0.0
            for _ in range(steps):
                self.flush.zero_()
                ev0.record(stream)
                g.replay()
                ev1.record(stream)
                ev1.synchronize()
                tot += ev0.elapsed_time(ev1)
            return tot
        full, rem = divmod(steps, self.nset)
        gf = self.graph(kind, self.nset) if full else None
        gr = self.graph(kind, rem) if rem else None
        ev0.record(stream)
        for _ in range(full):
            gf.replay()
        if gr is not None:
            gr.replay()
        ev1.record(stream)
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1)

    def l2_note(self) -> str:
        return l2_note_of(self.nset, self.cold, self.touched)


def l2_plan(d, pool, min_sets=4, max_sets=128):
    """Rotating buffer sets for L2-cold steps: (sets, cold, bytes touched per step).  Host arithmetic
    only (the reference arm states the same plan in its config)."""
    N = d["N"]
    Oh = (d["H"] + d["pad_top"] + d["pad_bottom"] - d["R"]) // d["stride_h"] + 1
    Ow = (d["W"] + d["pad_left"] + d["pad_right"] - d["S"]) // d["stride_w"] + 1
    rho = float((pool != 0).mean())
    x_b = 4 * N * d["C"] * d["H"] * d["W"]
    enc_b = 2 * 8 * rho * N * d["C"] * d["H"] * d["W"] + 4 * N * d["C"] * (3 + 2 * (d["W"] + 2))
    w_b = 4 * d["K"] * d["C"] * d["R"] * d["S"]
    y_b = 4 * N * d["K"] * Oh * Ow
    touched = x_b + enc_b + w_b + y_b          # per step (encode reads x, writes enc; conv reads enc, w)
    need = int(np.ceil(1.5 * L2_BYTES / touched))
    cold = need <= max_sets
    return (max(min_sets, min(need, max_sets)) if cold else min_sets), cold, touched


def l2_note_of(nset, cold, touched) -> str:
    if cold:
        return (f"inputs larger than L2: back-to-back steps over {nset} buffer sets, "
                f"~{nset * touched / 2**20:.0f} MiB touched per cycle (L2 126 MiB)")
    return f"L2 flushed between steps (2x-L2 write; {nset} sets would not exceed L2)"


def spc_out_hw(d):
    import paper_2104_08314_b200 as spc
    return spc.spc_output_dims(d)


def make_pool(c, rank: int = 0, distinct: int = 4):
    """Distinct seeded clustered-ReLU images of a config (each rank draws its own)."""
    d = c["desc"]
    nd = max(d["N"], distinct)
    return clustered_relu(nd, d["C"], d["H"], d["W"], c["density"], c["seed"] + 7919 * rank, c["dead_frac"],
                          c["zero_tile_frac"])


def fp32_peak(sm_max_mhz):
    return SM_COUNT * FP32_LANES * 2 * sm_max_mhz * 1e6 / 1e12   # TFLOP/s, derived


def measure_layer(name, d, pool, w, dev, stream, steps, hbm_gbs, p_fp32, im2col=True, cps=True):
    """One per-config row: encode / conv / step / CPS / im2col device times per launch (back to
    back over rotating sets), the conv's FP32 roofline fraction, the encoder's HBM fraction,
    the compression ratio and the exact NZE work."""
    import paper_2104_08314_b200 as spc
    R = Rotating(d, pool, w, dev)
    Oh, Ow = spc_out_hw(d)
    t = {k: R.timed(k, steps, stream) / steps * 1e3 for k in ("step", "encode", "conv")}
    if cps:
        t["cps_step"] = R.timed("cps", steps, stream) / steps * 1e3
    if im2col:
        t["im2col"] = R.timed("im2col", steps, stream) / steps * 1e3
    L0 = R.layers[0]
    L0.forward(R.xs[0], "cpo")
    pl_, dl_, il_ = L0.lengths()
    x0 = R.xs[0].cpu().numpy()
    macs = nze_macs(d, x0, Oh, Ow)
    flops = 2.0 * macs
    conv_bytes = 4 * (pl_ + dl_ + il_) + 8 * 2 * (d["N"] * d["C"] + 1) + 4 * d["K"] * d["C"] * d["R"] * d["S"] + \
        4 * d["N"] * d["K"] * Oh * Ow
    enc_bytes = 4 * x0.size + 4 * (pl_ + dl_ + il_) + 8 * 3 * (d["N"] * d["C"] + 1)
    s_im2col = d["N"] * Oh * Ow * d["C"] * d["R"] * d["S"]
    t_roof = max(conv_bytes / (hbm_gbs * 1e9), flops / (p_fp32 * 1e12))
    row = {"workload": name, "shape": {k: d[k] for k in d}, "density_measured": round(float((x0 != 0).mean()), 4),
           "encode_us": t["encode"], "conv_us": t["conv"], "step_us": t["step"],
           "dense_equiv_gflops": dense_flops(d, Oh, Ow) / (t["step"] * 1e-6) / 1e9,
           "conv_fp32_frac": t_roof / (t["conv"] * 1e-6), "conv_tflops_nze": flops / (t["conv"] * 1e-6) / 1e12,
           "encode_hbm_frac": enc_bytes / (t["encode"] * 1e-6) / 1e9 / hbm_gbs,
           "encode_gbs": enc_bytes / (t["encode"] * 1e-6) / 1e9,
           "cr_cpo": s_im2col / (pl_ + dl_ + il_), "nze_macs": macs, "l2": R.l2_note()}
    if cps:
        row["cps_step_us"] = t["cps_step"]
    if im2col:
        row["im2col_us"] = t["im2col"]
        row["im2col_gemm"] = spc.GEMM_NAMES[spc.spc_im2col_engine(d)]
        row["speedup_vs_im2col"] = t["im2col"] / t["step"]
    return row, R


def measure_extra(name, d, pool, w, dev, stream, steps, kinds):
    """Other encodings of the same layer, back to back over rotating sets: the CSCC baseline
    (the paper's comparison method) and the stride-aware layout; step us and CR vs S_im2col."""
    R = Rotating(d, pool, w, dev)
    Oh, Ow = spc_out_hw(d)
    s_im2col = d["N"] * Oh * Ow * d["C"] * d["R"] * d["S"]
    row = {"workload": name}
    for k in kinds:
        row[f"{k}_step_us"] = R.timed(k, steps, stream) / steps * 1e3
        L0 = R.layers[0]
        L0.forward(R.xs[0], k)
        import paper_2104_08314_b200 as spc
        p, a, i = spc.spc_encoding_lengths(L0.extra_encoding(k))
        row[f"cr_{k}"] = s_im2col / (p + a + i)
        row[f"{k}_ptr"] = p
    row["cpo_step_us"] = R.timed("step", steps, stream) / steps * 1e3
    L0 = R.layers[0]
    L0.forward(R.xs[0], "cpo")
    p, a, i = L0.lengths()
    row["cr_cpo"] = s_im2col / (p + a + i)
    row["cpo_ptr"] = p
    row["l2"] = R.l2_note()
    return row


def measure_fused_chain(dev, stream, steps, rank=0, kinds=("separate", "fused", "conv1", "conv1_fused", "encode2")):
    """NEXT-1 on the cfg4 chain (1x7 -> ReLU -> 7x1, BASELINE.json configs[3]): layer 1's conv
    emitting layer 2's CPO encoding (sparse_conv_encode_forward) against conv + a separate
    cpo_encode of the dense intermediate; both followed by layer 2's conv.  Back to back over
    rotating buffer sets (each set > L2 / NSET)."""
    import torch

    import paper_2104_08314_b200 as spc
    from paper_2104_08314_b200.layer import SparseConvLayer
    a, b = CONFIGS["cfg4a"], CONFIGS["cfg4b"]
    d1, d2 = a["desc"], b["desc"]
    pool = make_pool(a, rank)
    w1 = he_normal(d1["K"], d1["C"], 1, 7, a["seed"])
    w2 = he_normal(d2["K"], d2["C"], 7, 1, b["seed"] + 1)
    touched = 4 * (2 * pool[0].size * d1["N"] + w1.size + w2.size) + 8 * 0.5 * pool[0].size * d1["N"]
    nset = int(min(64, max(4, np.ceil(1.5 * L2_BYTES / touched))))
    sets = []
    for i in range(nset):
        idx = [(i + j) % pool.shape[0] for j in range(d1["N"])]
        x = torch.from_numpy(np.ascontiguousarray(pool[idx])).to(dev)
        L1 = SparseConvLayer(d1, torch.from_numpy(w1).to(dev), device=dev, relu=True)
        L2 = SparseConvLayer(d2, torch.from_numpy(w2).to(dev), device=dev)
        out = spc.alloc_encoding(d2, device=dev)
        fws = spc.alloc_fused_workspace(d1, device=dev)
        L1.encode(x)
        sets.append((x, L1, L2, out, fws))

    def run(kind, n):
        for i in range(n):
            x, L1, L2, out, fws = sets[i % nset]
            if kind == "separate":      # conv 1 (ReLU) -> encode y1 -> conv 2
                L1.conv()
                L2.encode(L1.y)
                L2.conv()
            elif kind == "fused":       # conv 1 emitting layer 2's encoding -> conv 2
                spc.sparse_conv_encode_forward(d1, L1.enc, L1.wp, L1.y, True, d2, out, fws)
                spc.sparse_conv_forward(d2, out, L2.wp, L2.y, False, L2.ws)
            elif kind == "conv1":
                L1.conv()
            elif kind == "conv1_fused":
                spc.sparse_conv_encode_forward(d1, L1.enc, L1.wp, L1.y, True, d2, out, fws)
            elif kind == "encode2":
                L2.encode(L1.y)
    res = {}
    for kind in kinds:
        run(kind, nset)
        torch.cuda.synchronize()
        g = sets[0][1].capture(lambda: run(kind, nset), warmup=1)
        reps = max(1, steps // nset)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        res[f"{kind}_us"] = e0.elapsed_time(e1) / (reps * nset) * 1e3
        del g
    if len(kinds) == 5:
        res["encoder_saved_us"] = res["conv1_us"] + res["encode2_us"] - res["conv1_fused_us"]
        res["chain_speedup"] = res["separate_us"] / res["fused_us"]
    res["workload"] = "cfg4 chain: 1x7 (pad 0,3) -> ReLU -> 7x1 (pad 3,0), 8x192x17x17"
    res["l2"] = f"back to back over {nset} buffer sets"
    res["fused_form"] = ("layer-1 conv epilogue emits per-column output row masks; 3 launches build layer 2's "
                         "CPO streams reading only the NZEs (no dense re-scan); bit-identical to cpo_encode")
    return res


# ---------------------------------------------------------------- cfg5 stack leg

def run_stack(args, world, rank, dev, hbm_gbs, p_fp32, mode="best_of_three", force=None, S=None):
    """cfg5: global batch args.stack_batch sharded over the ranks (strong scaling of this
    sub-metric).  The per-layer plan is selected offline ONCE on rank 0 and
    persisted to a plan file every rank reads (no collective carries it);
    force="cpo" runs the method on all 16 layers instead.  The 16 layers are one CUDA
    graph; then the one output gather.  Every layer's data exceeds L2 at this batch, so
    steps run back to back.  images/s = global batch / max over ranks of device time."""
    import tempfile

    import torch
    import torch.distributed as dist

    import paper_2104_08314_b200 as spc
    from paper_2104_08314_b200.stack import Cfg5Stack, gather_outputs, load_plan, save_plan, shard_range
    lo, hi = shard_range(args.stack_batch, world, rank)
    if S is None:
        S = Cfg5Stack(hi - lo, dev, rank=rank)
    names = [sp["name"] for sp in S.specs]
    if force:
        plan = [force] * len(S.layers)
        plan_src = f"forced: {force} on every layer"
    else:
        path = args.plan_file or os.path.join(tempfile.gettempdir(),
                                              f"spc_cfg5_plan_{mode}_{os.environ.get('MASTER_PORT', '0')}.json")
        if rank == 0 and not args.plan_file:
            S.select(mode)
            save_plan(path, names, S.plan, mode, S.select_times, [sp["density"] for sp in S.specs])
        if world > 1:
            dist.barrier()   # control plane only: the plan travels through the file
        plan = load_plan(path, names)
        plan_src = f"offline selection ({mode}) on rank 0, read from plan file {os.path.basename(path)}"
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
    # per-layer device time of the chosen algorithm (one graph per layer, back to back)
    layer_ms = []
    for L, x, algo in zip(S.layers, S.inputs, S.plan):
        g = L.capture(lambda L=L, x=x, algo=algo: L.forward(x, algo), warmup=1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(3):
            g.replay()
        e1.record(stream)
        torch.cuda.synchronize()
        layer_ms.append(e0.elapsed_time(e1) / 3)
        del g
    # roofline of the chosen plan (per-layer t_roof = max(bytes / HBM, FLOPs / peak of its engine))
    t_roof, t_roof_sparse = 0.0, 0.0
    layers = []
    for sp, L, algo, xb, lms in zip(S.specs, S.layers, S.plan, S.host_inputs, layer_ms):
        d = sp["desc"]
        Oh, Ow = L.Oh, L.Ow
        reps = (d["N"] + xb.shape[0] - 1) // xb.shape[0]
        x_bytes = 4 * d["N"] * d["C"] * d["H"] * d["W"]
        y_bytes = 4 * d["N"] * d["K"] * Oh * Ow
        w_bytes = 4 * d["K"] * d["C"] * d["R"] * d["S"]
        macs = nze_macs(dict(d, N=xb.shape[0]), xb, Oh, Ow) * reps * (d["N"] / (xb.shape[0] * reps))
        nnz = int((xb != 0).sum()) * d["N"] / xb.shape[0]
        enc_bytes = x_bytes + 8 * nnz + 8 * 3 * d["N"] * d["C"]
        tr_sparse = enc_bytes / (hbm_gbs * 1e9) + max((8 * nnz + w_bytes + y_bytes) / (hbm_gbs * 1e9),
                                                       2.0 * macs / (p_fp32 * 1e12))
        if algo == "im2col":
            low = 4 * d["N"] * d["C"] * d["R"] * d["S"] * Oh * Ow
            if spc.spc_im2col_engine(d) == spc.SPC_GEMM_TC_3XTF32:
                t_mma = 3 * dense_flops(d, Oh, Ow) / (tf32_peak() * 1e12)   # three TF32 products per MAC
            else:
                t_mma = dense_flops(d, Oh, Ow) / (p_fp32 * 1e12)
            tr = max((x_bytes + 2 * low + w_bytes + y_bytes) / (hbm_gbs * 1e9), t_mma)
        else:
            tr = tr_sparse
        t_roof += tr
        t_roof_sparse += tr_sparse
        from paper_2104_08314_b200.bounds import space_preselect
        rbar = float((xb != 0).mean())
        layers.append({"layer": sp["name"], "density": round(sp["density"], 4), "algo": algo,
                       "space_preselect_vs_im2col": space_preselect(d, rbar, "im2col"),
                       "device_ms": round(lms, 4), "roofline_frac": round(tr / (lms * 1e-3), 4),
                       "nze_gflop": round(2.0 * macs / 1e9, 3)})
    agree = sum(1 for L in layers if (L["space_preselect_vs_im2col"] == "cpo") == (L["algo"] in ("cpo", "cps")))
    res = {"workload": "cfg5 ResNet-50 3x3 stack (16 layers)", "global_batch": args.stack_batch,
           "preselect_vs_timed_plan": {"agree": agree, "layers": len(layers),
                                       "note": "zero-cost SI space pre-selector (CPO smaller than the im2col matrix: "
                                               "every 3x3 layer at every density) against the timed plan"},
           "per_rank_batch": hi - lo, "n_gpus": world, "mode": mode if not force else f"forced {force}",
           "plan_source": plan_src,
           "images_per_s": args.stack_batch / (t_tot * 1e-3), "ms_per_step": t_tot, "stack_ms": t_stack,
           "gather_ms": t_gather, "gather": "NCCL all_gather_into_tensor of the last layer's output" if world > 1
           else "none (1 GPU)", "steps": args.stack_steps, "scaling": "strong (global batch fixed)",
           "roofline_images_per_s": (hi - lo) / t_roof if t_roof > 0 else None,
           "roofline_frac": (t_roof * 1e3) / t_tot if t_tot > 0 else None,
           "roofline_model": "sum over layers of the chosen algorithm's bound: sparse = encode bytes / HBM + "
                             "max(compressed + weight + output bytes / HBM, NZE FLOPs / FP32 peak); im2col = "
                             "max(x + 2 x lowered + w + y bytes / HBM, dense FLOPs / FP32 peak (cuBLAS FP32) or "
                             "3 x dense FLOPs / TF32 tensor peak (tcgen05 3xTF32))",
           "plan": layers, "select_ms_per_sample": S.select_times if (rank == 0 and not force) else None,
           "gemm_per_layer": [spc.GEMM_NAMES[spc.spc_im2col_engine(sp["desc"])] for sp in S.specs],
           "inputs": "8 distinct seeded clustered-ReLU images per layer, tiled to the batch; every layer's data "
                     "exceeds L2 at this batch, steps back to back"}
    if force:
        res["sparse_roofline_images_per_s"] = (hi - lo) / t_roof_sparse
    return res, S


# ---------------------------------------------------------------- GPU leg

PER_CONFIG = ["cfg1", "cfg2", "cfg3", "cfg3s2", "cfg3@0.05", "cfg3@0.2", "cfg3@0.3", "cfg3@0.5", "cfg4a", "cfg4b"]


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
    hbm_gbs, sm_max_mhz, peak_src = load_peaks()
    p_fp32 = fp32_peak(sm_max_mhz)

    c = workload(args.workload)
    d = c["desc"]
    pool = make_pool(c, rank)                       # each rank draws its own images (weak scaling)
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    Oh, Ow = spc_out_hw(d)
    R = Rotating(d, pool, w, dev)
    g_step_full = R.graph("step", R.nset)           # capture before the timed region

    # --- main timed region (CPO encode + conv), barrier + sync on both sides, max over ranks
    for _ in range(max(1, args.warmup // R.nset + 1)):
        g_step_full.replay()
    R.timed("step", args.warmup, stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        t_ms = R.timed("step", args.steps, stream)
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

    # --- per-launch kernel durations (back to back over the same rotating sets, L2-cold):
    #     the rooflines use these averages
    k_steps = max(args.steps, 4 * R.nset)
    k_enc_ms = R.timed("encode", k_steps, stream) / k_steps
    k_conv_ms = R.timed("conv", k_steps, stream) / k_steps
    t_cps_ms = R.timed("cps", args.steps, stream) / args.steps
    t_i2c_ms = R.timed("im2col", args.steps, stream) / args.steps

    L0 = R.layers[0]
    L0.forward(R.xs[0], "cpo")
    import paper_2104_08314_b200 as spc
    conv_kernel = spc.CONV_KERNELS.get(spc.spc_last_conv_kernel(), "?")   # the headline conv's kernel
    pl_, dl_, il_ = L0.lengths()
    L0.forward(R.xs[0], "cps")
    ps_, ds_, is_ = L0.lengths()
    L0.forward(R.xs[0], "cpo")
    x0 = R.xs[0].cpu().numpy()
    s_im2col = d["N"] * Oh * Ow * d["C"] * d["R"] * d["S"]
    side = 3 * (d["N"] * d["C"] + 1) * 2   # int64 side tables in 4-byte elements
    cr_cpo = s_im2col / (pl_ + dl_ + il_)
    cr_cps = s_im2col / (ps_ + ds_ + is_)

    # --- roofline of the dominant kernel (measured per-launch averages)
    macs = nze_macs(d, x0, Oh, Ow)
    conv_bytes = 4 * (pl_ + dl_ + il_) + 8 * 2 * (d["N"] * d["C"] + 1) + 4 * w.size + 4 * d["N"] * d["K"] * Oh * Ow
    enc_bytes = 4 * x0.size + 4 * (pl_ + dl_ + il_) + 8 * 3 * (d["N"] * d["C"] + 1)
    conv_s, enc_s = k_conv_ms * 1e-3, k_enc_ms * 1e-3
    conv_flops = 2.0 * macs
    t_roof_conv = max(conv_bytes / (hbm_gbs * 1e9), conv_flops / (p_fp32 * 1e12))
    conv_bound = "alu" if conv_flops / (p_fp32 * 1e12) >= conv_bytes / (hbm_gbs * 1e9) else "hbm"
    traffic, traffic_src = None, None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            tj = json.load(open(tfile))
            traffic = tj.get(args.workload, {}).get("sparse_conv" if conv_s >= enc_s else "encode")
            traffic_src = tj.get("_source")
        except Exception:
            traffic = None
    if conv_s >= enc_s:
        roof = {"kernel": f"sparse conv ({conv_kernel})", "bound": conv_bound,
                "achieved": conv_flops / conv_s / 1e12 if conv_bound == "alu" else conv_bytes / conv_s / 1e9,
                "peak": p_fp32 if conv_bound == "alu" else hbm_gbs, "unit": "TFLOP/s" if conv_bound == "alu" else "GB/s",
                "frac": t_roof_conv / conv_s, "traffic": traffic, "traffic_source": traffic_src,
                "peak_source": "derived: 148 SMs x 128 FP32 lanes x 2 x max SM clock (tools/ffma_peak.cu measured "
                               "72.6 TFLOP/s)" if conv_bound == "alu" else peak_src,
                "algorithmic_flops_per_launch": conv_flops, "algorithmic_bytes_per_launch": conv_bytes,
                "launch_us": conv_s * 1e6,
                "timing": f"mean launch duration over {k_steps} back-to-back launches (CUDA events on the "
                          f"launching stream), {R.l2_note()}"}
    else:
        roof = {"kernel": "encode_kernel", "bound": "hbm", "achieved": enc_bytes / enc_s / 1e9, "peak": hbm_gbs,
                "unit": "GB/s", "frac": enc_bytes / enc_s / 1e9 / hbm_gbs, "traffic": traffic,
                "traffic_source": traffic_src, "peak_source": peak_src, "algorithmic_bytes_per_launch": enc_bytes,
                "launch_us": enc_s * 1e6}

    # --- end to end through the public API with host buffers: pinned H2D of the
    # input, encode + conv, D2H of the output, all inside the timed region
    xg, y = R.xs[0], L0.y
    xh = torch.from_numpy(x0).pin_memory()
    yh = torch.empty(y.shape, dtype=torch.float32).pin_memory()

    def e2e_step():
        xg.copy_(xh, non_blocking=True)
        L0.forward(xg, "cpo")
        yh.copy_(y, non_blocking=True)
    g_e2e = L0.capture(e2e_step)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        g_e2e.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_serial_ms = e0.elapsed_time(e1)

    # Pipelined form of the same steps (what a serving loop does): NB buffer sets; per step,
    # H2D on one stream, encode + conv on a second, D2H on a third, so step i's copies
    # overlap the neighbouring steps' compute.  One graph holds PIPE steps.
    PIPE = int(os.environ.get("BENCH_E2E_PIPE", "64"))   # steps per graph (fill / drain amortised)
    NB = min(len(R.layers), int(os.environ.get("BENCH_E2E_NB", "2")))   # buffer sets in flight
    Ls = [R.layers[b] for b in range(NB)]
    xgs = [R.xs[b] for b in range(NB)]
    yhs = [yh] + [torch.empty(y.shape, dtype=torch.float32).pin_memory() for _ in range(NB - 1)]
    s_h, s_c, s_d = (torch.cuda.Stream(device=dev) for _ in range(3))
    ev_h = [torch.cuda.Event() for _ in range(PIPE)]
    ev_c = [torch.cuda.Event() for _ in range(PIPE)]
    ev_d = [torch.cuda.Event() for _ in range(PIPE)]

    def pipeline():
        cs = torch.cuda.current_stream()
        for st_ in (s_h, s_c, s_d):
            st_.wait_stream(cs)
        for i in range(PIPE):
            b = i % NB
            with torch.cuda.stream(s_h):
                if i >= NB:
                    s_h.wait_event(ev_c[i - NB])     # xg[b] free: step i-NB's encode read it
                xgs[b].copy_(xh, non_blocking=True)
                ev_h[i].record(s_h)
            with torch.cuda.stream(s_c):
                s_c.wait_event(ev_h[i])
                if i >= NB:
                    s_c.wait_event(ev_d[i - NB])     # y[b] free: step i-NB's D2H read it
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
    e0.record(stream)
    for _ in range(reps):
        g_pipe.replay()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) * args.steps / (reps * PIPE)   # per-step mean, scaled to K steps
    if world > 1:
        tt = torch.tensor([e2e_ms, e2e_serial_ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_ms, e2e_serial_ms = float(tt[0].item()), float(tt[1].item())
    e2e_val = flops_step * args.steps * world / (e2e_ms * 1e-3) / 1e9
    R_note = R.l2_note()
    del R, g_step_full, g_e2e, g_pipe
    torch.cuda.empty_cache()

    # --- per-config rows (rank 0 draws them; each row is its own rotating buffer set)
    rows = []
    if not args.no_configs:
        y4a = None
        for name in PER_CONFIG:
            base, _, dens = name.partition("@")
            cc = dict(workload(base))
            if dens:
                cc["density"] = float(dens)
            dd = cc["desc"]
            if base == "cfg4b":
                if y4a is None:
                    continue
                pool_c = y4a            # ReLU(cfg4a output): the intermediate re-sparsified by ReLU
            else:
                pool_c = make_pool(cc, rank)
            wc = he_normal(dd["K"], dd["C"], dd["R"], dd["S"], cc["seed"] + (1 if base == "cfg4b" else 0))
            row, Rc = measure_layer(name, dd, pool_c, wc, dev, stream, args.config_steps, hbm_gbs, p_fp32)
            if base == "cfg4a":
                L = Rc.layers[0]
                L.relu = True
                L.forward(Rc.xs[0], "cpo")
                y4a = L.y.cpu().numpy()
                L.relu = False
            rows.append(row)
            del Rc
            torch.cuda.empty_cache()

    extras = None
    if not args.no_configs:
        extras = {"fused_chain_cfg4": measure_fused_chain(dev, stream, args.config_steps, rank), "cscc": [],
                  "stride_aware": []}
        for name in ("cfg2", "cfg3", "cfg3s2", "cfg4a"):
            cc = workload(name)
            dd = cc["desc"]
            extras["cscc"].append(measure_extra(name, dd, make_pool(cc, rank),
                                                he_normal(dd["K"], dd["C"], dd["R"], dd["S"], cc["seed"]), dev, stream,
                                                args.config_steps, ["cscc"]))
            torch.cuda.empty_cache()
        for name in ("cfg3s2", "cfg5L3", "cfg5L7", "cfg5L13"):
            cc = workload(name)
            dd = cc["desc"]
            extras["stride_aware"].append(measure_extra(name, dd, make_pool(cc, rank),
                                                        he_normal(dd["K"], dd["C"], dd["R"], dd["S"], cc["seed"]),
                                                        dev, stream, args.config_steps, ["cpo_sa"]))
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and not args.no_cpu:
        t, n, f = oracle_time(d, pool[:d["N"]], w, budget_s=args.cpu_budget)
        cpu = {"value": f / t / 1e9, "unit": "GFLOP/s", "cores": 1, "kind": "oracle",
               "host_cpus": os.cpu_count(), "cpu_model": cpu_model(),
               "sample": f"{n} image(s) of {args.workload}: oracle CPO encode + Alg. 2 conv, single thread, FP64"}
        cpu["legs"] = oracle_legs(d, pool[:d["N"]], w)
        t2, n2, f2, thr = oracle_time_threads(d, pool[:d["N"]], w, args.cpu_budget, os.cpu_count() or 1)
        cpu["all_cores"] = {"value": f2 / t2 / 1e9, "unit": "GFLOP/s", "cores": thr,
                            "sample": f"{n2} image(s): encode on one thread, Alg. 2 over {thr} output-channel "
                                      "slices in parallel threads"}

    stack = stack_cpo = None
    if not args.no_stack:
        stack, S = run_stack(args, world, rank, dev, hbm_gbs, p_fp32, mode=args.stack_mode)
        stack_cpo, _ = run_stack(args, world, rank, dev, hbm_gbs, p_fp32, force="cpo", S=S)
        if rank == 0 and not args.no_cpu:
            import oracle
            oracle.build()
            t_cpu = 0.0
            for sp, xb, wl in zip(S.specs, S.host_inputs, S.weights):
                t, n, _ = oracle_time(dict(sp["desc"], N=2), xb[:2], wl, budget_s=1e9)
                t_cpu += t
            stack["cpu_baseline"] = {"value": 2 / t_cpu, "unit": "images/s", "cores": 1, "kind": "oracle",
                                     "sample": "2 images through all 16 layers: oracle CPO encode + Alg. 2 conv, "
                                               "single thread, FP64"}
        del S
        torch.cuda.empty_cache()

    if world > 1:
        dist.barrier()
    if rank == 0:
        us = lambda ms: 1e3 * ms  # noqa: E731
        line = {
            "metric": METRIC,
            "value": value, "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tmax / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": args.workload, **{k: d[k] for k in d}, "density": c["density"],
                       "dead_frac": c["dead_frac"], "zero_tile_frac": c["zero_tile_frac"],
                       "l2": R_note, "global_batch": d["N"] * world},
            "layer_us": {"cpo_step": us(tmax / args.steps), "cpo_encode": us(k_enc_ms), "cpo_conv": us(k_conv_ms),
                         "cps_step": us(t_cps_ms), "im2col_step": us(t_i2c_ms)},
            "kernel_us": {"timing": "mean per launch, back-to-back launches over the rotating L2-cold buffer sets",
                          "cpo_conv": us(k_conv_ms), "cpo_encode": us(k_enc_ms)},
            "im2col": {"value": flops_step / (t_i2c_ms * 1e-3) / 1e9, "unit": "GFLOP/s",
                       "gemm": spc.GEMM_NAMES[spc.spc_im2col_engine(d)]},
            "speedup_vs_im2col": t_i2c_ms / (tmax / args.steps),
            "cr": {"cpo": cr_cpo, "cps": cr_cps, "cpo_with_side_tables": s_im2col / (pl_ + dl_ + il_ + side),
                   "ptr": pl_, "da": dl_, "in_cpo": il_, "in_cps": is_, "S_im2col": s_im2col},
            "nze_macs": macs, "density_measured": float((x0 != 0).mean()),
            "roofline": roof,
            "roofline_encode": {"bound": "hbm", "achieved": enc_bytes / enc_s / 1e9, "peak": hbm_gbs,
                                "unit": "GB/s", "frac": enc_bytes / enc_s / 1e9 / hbm_gbs},
            "e2e": {"value": e2e_val, "unit": "GFLOP/s", "h2d_bytes_per_step": int(4 * x0.size),
                    "d2h_bytes_per_step": int(4 * d["N"] * d["K"] * Oh * Ow), "ms_per_step": e2e_ms / args.steps,
                    "form": f"pipelined: H2D / encode+conv / D2H on three streams, {PIPE} steps per graph, {NB} buffer sets "
                            "(fill and drain included)",
                    "serial": {"value": flops_step * args.steps * world / (e2e_serial_ms * 1e-3) / 1e9,
                               "ms_per_step": e2e_serial_ms / args.steps,
                               "form": "one step per graph: H2D, encode, conv, D2H in sequence"}},
            "gpu_launches": 2 * args.steps,
            "clocks": clk.summary(),
            "cpu_baseline": cpu,
            "configs": rows,
            "extras": extras,
            "stack": stack,
            "stack_cpo": stack_cpo,
            "version": spc.spc_version(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--no-configs", action="store_true", help="skip the per-config rows")
    ap.add_argument("--config-steps", type=int, default=200)
    ap.add_argument("--plan-file", default="", help="read the cfg5 plan from this file (skip selection)")
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
