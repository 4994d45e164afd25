"""Zero-cost space pre-selector from the SI's closed-form bounds.

Argument marshalling only: the arithmetic lives behind the C ABI (spc_space_bound,
spc_cscc_q_bound, spc_space_preselect in include/spconv.h); the oracle's independent copy is
oracle/sizes.py, and tests/test_bounds.py compares the two.
"""
from __future__ import annotations

from . import binding as B

_VS = {"im2col": B.SPC_SPACE_VS_IM2COL, "mec": B.SPC_SPACE_VS_MEC, "cscc": B.SPC_SPACE_VS_CSCC}


def rho_space_bound(d: dict, vs: str = "im2col", rho_hat_bar: float = 0.0) -> float:
    """Largest average density at which CPO is no larger than `vs` ("im2col", "mec", "cscc")."""
    return B.spc_space_bound(d, _VS[vs], rho_hat_bar)


def cscc_q_bound(d: dict) -> float:
    """Q(rho_hat): least average lowered-matrix density with a non-empty CSCC bound."""
    return B.spc_cscc_q_bound(d)


def space_preselect(d: dict, rho_bar: float, vs: str = "im2col", rho_hat_bar: float = 0.0) -> str:
    """favour-space pre-selection without timing: 'cpo' inside P(rho), else the dense method."""
    return B.ALGO_NAMES[B.spc_space_preselect(d, _VS[vs], rho_bar, rho_hat_bar)]
