"""cfg5 (BASELINE.json configs[4]): the ResNet-50-shaped stack of the 16 non-pointwise
3x3 layers, batch sharded over GPUs, with the paper's offline per-layer selection
between CPO, CPS and im2col (§3.5) and one output gather at the end.

Host-side orchestration only: every layer runs through the C ABI (libspconv.so);
PyTorch provides device memory, streams, CUDA graphs and torch.distributed.

Multi-GPU: images are independent, so rank r owns the contiguous
image range shard_range(N, world, r) and runs the whole stack on it with no
exchange; the per-layer plan is chosen once (rank 0) and broadcast; the final
layer's outputs are gathered with one collective (NCCL over NVLink on GPUs, gloo
in the CPU tests).
"""
from __future__ import annotations

import json

import numpy as np
import torch

from . import binding as B
from .layer import ALGOS, SparseConvLayer

MODES = {"favour_time": B.SPC_FAVOUR_TIME, "favour_space": B.SPC_FAVOUR_SPACE,
         "best_of_three": B.SPC_BEST_OF_THREE}


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous image range of `rank` (sizes differ by at most one)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def broadcast_plan(plan: list[str] | None, src: int = 0) -> list[str]:
    """Rank `src` decides the per-layer algorithms; every rank gets the same list
    (control plane only: a pickled list of strings)."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return list(plan)
    box = [plan if dist.get_rank() == src else None]
    dist.broadcast_object_list(box, src=src)
    return list(box[0])


def gather_outputs(y: torch.Tensor, n_per_rank: list[int]) -> torch.Tensor:
    """The one data-path collective: all ranks' final outputs [n_r, ...] -> [sum n_r, ...]
    (in rank order) on every rank.  Ranks may hold different image counts."""
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return y
    world = dist.get_world_size()
    nmax = max(n_per_rank)
    pad = torch.zeros((nmax,) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
    pad[:y.shape[0]].copy_(y)
    if dist.get_backend() == "nccl":
        out = torch.empty((world * nmax,) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
        dist.all_gather_into_tensor(out, pad)
        parts = list(out.split(nmax))
    else:
        parts = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(parts, pad)
    return torch.cat([p[:n] for p, n in zip(parts, n_per_rank)])


def save_plan(path: str, layers: list[str], plan: list[str], mode: str, times_ms=None, density=None) -> None:
    """Persist a per-layer plan (the offline selection's result) so that ranks
    read it instead of re-selecting: written atomically (tmp + rename)."""
    import os
    doc = {"format": "spconv-b200 plan v1", "mode": mode, "layers": list(layers), "plan": list(plan),
           "select_times_ms": times_ms, "density": density}
    tmp = f"{path}.tmp{os.getpid()}"
    with open(tmp, "w") as f:
        json.dump(doc, f)
    os.replace(tmp, path)


def load_plan(path: str, layers: list[str] | None = None) -> list[str]:
    """Read a plan file written by save_plan; checks the layer names when given."""
    with open(path) as f:
        doc = json.load(f)
    if doc.get("format") != "spconv-b200 plan v1":
        raise ValueError(f"{path}: not a plan file")
    if layers is not None and list(doc["layers"]) != list(layers):
        raise ValueError(f"{path}: plan is for layers {doc['layers']}")
    plan = list(doc["plan"])
    if any(a not in ALGOS for a in plan):
        raise ValueError(f"{path}: bad algorithm in {plan}")
    return plan


def tile_images(base: np.ndarray, n: int) -> np.ndarray:
    """Fill a batch of n images by repeating `base` [b, C, H, W] (b distinct seeded
    images per layer; DESIGN.md §4 input recipe for the cfg5 stack)."""
    reps = (n + base.shape[0] - 1) // base.shape[0]
    return np.ascontiguousarray(np.concatenate([base] * reps, axis=0)[:n])


class Cfg5Stack:
    """The 16 layers of cfg5 for one rank's shard of the batch.  Each layer's input is
    generated independently; weights are He-normal from the
    layer seed (identical on every rank)."""

    def __init__(self, batch: int, device, seed: int = 105, distinct: int = 8, rank: int = 0):
        from synth import cfg5_layers, clustered_relu, he_normal
        self.device = torch.device(device)
        self.specs = cfg5_layers(batch=batch, seed=seed)
        self.layers: list[SparseConvLayer] = []
        self.inputs: list[torch.Tensor] = []
        self.host_inputs: list[np.ndarray] = []
        self.weights: list[np.ndarray] = []
        for sp in self.specs:
            d = sp["desc"]
            nb = min(distinct, batch)
            base = clustered_relu(nb, d["C"], d["H"], d["W"], sp["density"], sp["seed"] + 7919 * rank)
            x = tile_images(base, batch)
            w = he_normal(d["K"], d["C"], d["R"], d["S"], sp["seed"])
            self.host_inputs.append(base)
            self.weights.append(w)
            self.inputs.append(torch.from_numpy(x).to(self.device))
            self.layers.append(SparseConvLayer(d, torch.from_numpy(w).to(self.device), device=self.device))
        self.plan: list[str] = ["cpo"] * len(self.layers)
        self.select_times: list[list[float]] = []

    # ---- offline selection (M = 5 sample maps, distinct from the measured ones)
    def select(self, mode: str = "best_of_three", M: int = 5, reps: int = 2, select_seed: int = 1501,
               distinct: int = 2) -> list[str]:
        from synth import clustered_relu
        plan, times = [], []
        for i, (sp, L) in enumerate(zip(self.specs, self.layers)):
            d = sp["desc"]
            samples = []
            for m in range(M):
                base = clustered_relu(min(distinct, d["N"]), d["C"], d["H"], d["W"], sp["density"],
                                      select_seed + m + 100 * i)
                samples.append(tile_images(base, d["N"]))
            s = torch.from_numpy(np.stack(samples)).to(self.device)
            ws = torch.empty(B.spc_select_ws_bytes(d), dtype=torch.uint8, device=self.device)
            algo, t = B.select_layer_algo(d, s, M, L.w, MODES[mode], reps, ws)
            del ws
            plan.append(B.ALGO_NAMES[algo])
            times.append([float(v) for v in t])
            del s
        self.plan, self.select_times = plan, times
        return plan

    def set_plan(self, plan: list[str]):
        if len(plan) != len(self.layers) or any(a not in ALGOS for a in plan):
            raise ValueError(f"bad plan {plan}")
        self.plan = list(plan)

    def forward(self) -> torch.Tensor:
        """All 16 layers with the current plan; returns the last layer's output."""
        y = None
        for L, x, algo in zip(self.layers, self.inputs, self.plan):
            y = L.forward(x, algo)
        return y

    def capture(self) -> torch.cuda.CUDAGraph:
        return self.layers[0].capture(self.forward)

    def replay(self, times_ms: list[list[float]], mode: str = "best_of_three") -> list[str]:
        """The plan from RECORDED per-layer times {im2col, CPO, CPS} (SPEC.md:741 replay):
        the same argmin / tie rule as select_layer_algo, through the C ABI, no GPU work."""
        if len(times_ms) != len(self.layers):
            raise ValueError("one time triple per layer")
        plan = [B.ALGO_NAMES[B.spc_select_from_times(t, L.sparse_ok and t[1] >= 0 and t[2] >= 0, MODES[mode])]
                for t, L in zip(times_ms, self.layers)]
        self.plan, self.select_times = plan, [list(map(float, t)) for t in times_ms]
        return plan

    def plan_json(self) -> str:
        return json.dumps({"layers": [sp["name"] for sp in self.specs], "plan": self.plan,
                           "density": [sp["density"] for sp in self.specs],
                           "select_times_ms": self.select_times})
