"""GPU-test helpers: run the library on a layer and fetch its streams."""
from __future__ import annotations

import numpy as np
import torch

import paper_2104_08314_b200 as spc


class GpuLayer:
    """Owns the device buffers of one conv layer on the GPU path."""

    def __init__(self, d: dict, w: np.ndarray | None = None, caps=None):
        self.d = d
        self.enc = spc.alloc_encoding(d, caps=caps)
        self.ws = spc.alloc_workspace(d)
        Oh, Ow = spc.out_hw(d)
        self.y = torch.empty((d["N"], d["K"], Oh, Ow), dtype=torch.float32, device="cuda")
        if w is not None:
            self.set_weights(w)

    def set_weights(self, w: np.ndarray):
        self.w = torch.from_numpy(np.ascontiguousarray(w)).cuda()
        self.wp = torch.empty_like(self.w).reshape(-1)
        spc.spc_pack_weights(self.d, self.w, self.wp)

    def encode(self, x: torch.Tensor, cps: bool = False):
        (spc.cps_encode if cps else spc.cpo_encode)(self.d, x, self.enc, self.ws)
        return self

    def streams(self) -> dict:
        p, a, i = spc.spc_encoding_lengths(self.enc)
        e = self.enc
        return dict(ptr=e.ptr[:p].cpu().numpy(), da=e.da[:a].cpu().numpy(), inn=e.inn[:i].cpu().numpy(),
                    chan_ptr_off=e.chan_ptr_off.cpu().numpy(), chan_nz_off=e.chan_nz_off.cpu().numpy(),
                    chan_in_off=e.chan_in_off.cpu().numpy())

    def conv(self, relu: bool = False) -> torch.Tensor:
        spc.sparse_conv_forward(self.d, self.enc, self.wp, self.y, relu, self.ws)
        return self.y

    def im2col(self, x: torch.Tensor, relu: bool = False) -> torch.Tensor:
        Oh, Ow = spc.out_hw(self.d)
        d = self.d
        L = spc.alloc_im2col_workspace(d)
        y = torch.empty_like(self.y)
        spc.im2col_conv_forward(d, x, self.w, y, relu, L)
        return y


def assert_streams_equal(gpu: dict, ref: dict, what: str = ""):
    for k in ("ptr", "inn", "chan_ptr_off", "chan_nz_off", "chan_in_off"):
        a, b = gpu[k], ref[k]
        assert a.shape == b.shape, f"{what} {k}: length {a.shape} vs oracle {b.shape}"
        if not np.array_equal(a, b):
            bad = np.nonzero(a != b)[0]
            raise AssertionError(f"{what} {k}: {bad.size} mismatches, first at {bad[:5]}: "
                                 f"gpu {a[bad[:5]]} oracle {b[bad[:5]]}")
    # DA: bit-exact copies of the input
    assert gpu["da"].shape == ref["da"].shape, f"{what} da length"
    assert np.array_equal(gpu["da"].view(np.int32), ref["da"].view(np.int32)), f"{what} da bits"
