"""Replayable per-layer selection (§3.5; SPEC.md:657 argmin on the profiling
data, :741 replay from recorded profiles): spc_select_from_times (host-only C ABI, no GPU)
is pinned against a plain-Python argmin with the tie rule of reading A24 on the timings the
round-1 crossover sweep recorded on a B200 (profiles/r01_crossover.json), and the plan it
yields never takes longer than either pure strategy."""
import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MODES = {0: ("im2col", "cpo"), 1: ("im2col", "cps"), 2: ("im2col", "cpo", "cps")}
FOOTPRINT_RANK = {"cps": 0, "cpo": 1, "im2col": 2}                                    # A24: smaller first
CODE = {"im2col": 0, "cpo": 1, "cps": 2}


@pytest.fixture(scope="module")
def lib():
    from paper_2104_08314_b200 import build
    build.build()
    import paper_2104_08314_b200 as p
    return p


def py_argmin(times: dict, mode: int) -> str:
    cands = MODES[mode]
    return min(cands, key=lambda a: (times[a], FOOTPRINT_RANK[a]))


def recorded_profiles():
    out = []
    for f in ("r01_crossover.json", "r01_crossover_catalog.json"):
        data = json.load(open(os.path.join(ROOT, "profiles", f)))
        for layer in data["layers"]:
            for pt in layer["sweep"]:
                for eng, t_i2c in layer["im2col_us"].items():
                    if t_i2c is None or pt.get("cpo_us") is None or pt.get("cps_us") is None:
                        continue
                    out.append((layer["workload"], pt["rho"], eng,
                                {"im2col": float(t_i2c), "cpo": float(pt["cpo_us"]), "cps": float(pt["cps_us"])}))
    return out


def test_replay_equals_python_argmin_on_recorded_profiles(lib):
    recs = recorded_profiles()
    assert len(recs) > 300
    for wl, rho, eng, t in recs:
        for mode in (0, 1, 2):
            got = lib.spc_select_from_times([t["im2col"], t["cpo"], t["cps"]], True, mode)
            want = py_argmin(t, mode)
            assert got == CODE[want], (wl, rho, eng, mode, t)
            # the plan is never slower than either pure strategy of the mode
            assert t[lib.ALGO_NAMES[got]] <= min(t[a] for a in MODES[mode])


def test_ties_prefer_the_smaller_footprint(lib):
    assert lib.spc_select_from_times([5.0, 5.0, 5.0], True, 2) == lib.SPC_ALGO_CPS
    assert lib.spc_select_from_times([5.0, 5.0, 5.0], True, 0) == lib.SPC_ALGO_CPO
    assert lib.spc_select_from_times([5.0, 6.0, 5.0], True, 1) == lib.SPC_ALGO_CPS
    assert lib.spc_select_from_times([4.0, 5.0, 5.0], True, 2) == lib.SPC_ALGO_IM2COL
    assert lib.spc_select_from_times([5.0, 4.0, 4.0], True, 2) == lib.SPC_ALGO_CPS


def test_sparse_not_ok_routes_to_im2col_and_rejects_bad_times(lib):
    assert lib.spc_select_from_times([9.0, -1.0, -1.0], False, 2) == lib.SPC_ALGO_IM2COL
    with pytest.raises(lib.SpcError):
        lib.spc_select_from_times([1.0, -1.0, 2.0], True, 2)
    with pytest.raises(lib.SpcError):
        lib.spc_select_from_times([float("nan"), 1.0, 2.0], True, 0)
    with pytest.raises(lib.SpcError):
        lib.spc_select_from_times([1.0, 1.0, 1.0], True, 7)


def test_output_dims_floor_rule(lib):
    """reading A14: floor((I + pads - K) / s) + 1 (56 + 2 at s = 2 -> 28, 14 + 2 -> 7)."""
    from synth import layer_desc
    assert lib.spc_output_dims(layer_desc(1, 4, 56, 56, 4, 3, 3, 2, 2, 1, 1, 1, 1)) == (28, 28)
    assert lib.spc_output_dims(layer_desc(1, 4, 14, 14, 4, 3, 3, 2, 2, 1, 1, 1, 1)) == (7, 7)
    assert lib.spc_output_dims(layer_desc(1, 4, 17, 17, 4, 1, 7, 1, 1, 0, 0, 3, 3)) == (17, 17)
    assert lib.spc_output_dims(layer_desc(1, 4, 8, 8, 4, 4, 4, 1, 1, 0, 0, 0, 0)) == (5, 5)
