"""Layer-level convenience API over the C ABI: one conv layer's buffers, its
three algorithms (im2col, CPO, CPS) and CUDA-graph capture of a step.

All arithmetic runs in libspconv.so; this module only allocates device memory
with PyTorch and sequences the C calls.
"""
from __future__ import annotations

import torch

from . import binding as B

ALGOS = {"im2col": B.SPC_ALGO_IM2COL, "cpo": B.SPC_ALGO_CPO, "cps": B.SPC_ALGO_CPS}
# also runnable through forward(): the paper's comparison method and the stride-aware layout
EXTRA = ("cscc", "cpo_sa")


class SparseConvLayer:
    """Buffers of one layer: encoding capacity, workspace, packed weights, output,
    and (lazily) the im2col lowered-matrix workspace."""

    def __init__(self, desc: dict, w: torch.Tensor, device=None, relu: bool = False):
        self.d = dict(desc)
        self.device = torch.device(device) if device is not None else w.device
        self.w = w.to(self.device).contiguous()
        self.relu = relu
        self.Oh, self.Ow = B.out_hw(self.d)
        self.y = torch.empty((self.d["N"], self.d["K"], self.Oh, self.Ow), dtype=torch.float32, device=self.device)
        self.sparse_ok = True
        try:
            self.enc = B.alloc_encoding(self.d, device=self.device)
            self.ws = B.alloc_workspace(self.d, device=self.device)
        except B.SpcError:
            self.sparse_ok = False
            self.enc = self.ws = None
        self.wp = torch.empty_like(self.w).reshape(-1)
        B.spc_pack_weights(self.d, self.w, self.wp)
        self._lowered = None
        self._enc_x = {}     # lazily allocated encodings of the extra algorithms

    @property
    def lowered(self) -> torch.Tensor:
        if self._lowered is None:
            # lowered matrix + (tcgen05 engine) the once-per-call split of the weights
            self._lowered = B.alloc_im2col_workspace(self.d, device=self.device)
        return self._lowered

    # -- the three algorithms (asynchronous on the current stream)
    def encode(self, x: torch.Tensor, algo: str = "cpo"):
        (B.cps_encode if algo == "cps" else B.cpo_encode)(self.d, x, self.enc, self.ws)

    def conv(self) -> torch.Tensor:
        B.sparse_conv_forward(self.d, self.enc, self.wp, self.y, self.relu, self.ws)
        return self.y

    def extra_encoding(self, algo: str) -> B.Encoding:
        if algo not in self._enc_x:
            self._enc_x[algo] = (B.alloc_cscc_encoding(self.d, device=self.device) if algo == "cscc"
                                 else B.alloc_strided_encoding(self.d, device=self.device))
        return self._enc_x[algo]

    def forward(self, x: torch.Tensor, algo: str = "cpo") -> torch.Tensor:
        if algo == "cscc":           # CSCC baseline (SI Alg. 5 / 6)
            e = self.extra_encoding(algo)
            B.cscc_encode(self.d, x, e)
            B.cscc_conv_forward(self.d, e, self.wp, self.y, self.relu)
            return self.y
        if algo == "cpo_sa":         # stride-aware CPO layout (reading A32)
            e = self.extra_encoding(algo)
            B.cpo_encode_strided(self.d, x, e, self.ws)
            B.sparse_conv_forward(self.d, e, self.wp, self.y, self.relu, self.ws)
            return self.y
        if algo == "im2col" or not self.sparse_ok:
            B.im2col_conv_forward(self.d, x, self.w, self.y, self.relu, self.lowered)
            return self.y
        self.encode(x, algo)
        return self.conv()

    def lengths(self) -> tuple[int, int, int]:
        return B.spc_encoding_lengths(self.enc)

    def capture(self, fn, warmup: int = 2) -> torch.cuda.CUDAGraph:
        """CUDA-graph capture of `fn()` (a sequence of this layer's calls on static
        buffers).  Replaying the graph launches the same kernels with no host work."""
        s = torch.cuda.Stream(device=self.device)
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            for _ in range(warmup):
                fn()
        torch.cuda.current_stream(self.device).wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        return g
