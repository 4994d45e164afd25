"""Pins of the oracle against the values the paper prints for its Fig. 1 example.

Each assertion names the sentence of PAPER.md it checks (see tests/golden/fig1.json).
"""
import numpy as np
import pytest

from helpers import load_fig1


def test_fig1_cpo_streams(oracle_mod):
    d, x, exp = load_fig1()
    enc = oracle_mod.encode(d, x, cps=False)
    assert enc["ptr"].tolist() == exp["ptr"]
    assert enc["da"].tolist() == exp["da"]
    assert enc["inn"].tolist() == exp["in_cpo"]
    # overlap2 block exactly as PAPER.md:138 states it
    assert enc["ptr"][3:9].tolist() == [2, 5, -1, -1, 5, -1]
    assert enc["da"][:5].tolist() == [10, 20, 30, 40, 50]
    assert enc["inn"][:5].tolist() == [5, 9, 13, 17, 21]


def test_fig1_cps_streams(oracle_mod):
    d, x, exp = load_fig1()
    enc = oracle_mod.encode(d, x, cps=True)
    assert enc["ptr"].tolist() == exp["ptr"]          # CPS executes CPO for ptr
    assert enc["da"].tolist() == exp["da"]
    assert enc["inn"].tolist() == exp["in_cps"]
    assert [7, 14] == enc["inn"][6:8].tolist()         # PAPER.md:319 {3,7,11,15} -> {7,14}
    assert enc["inn"][5] == -23                        # PAPER.md:319 "-23 as a singleton"


def test_fig1_sizes(oracle_mod):
    d, x, exp = load_fig1()
    assert oracle_mod.im2col(d, x).size == exp["S_im2col"] == oracle_mod.S_im2col(d)
    assert oracle_mod.mec_lower(d, x).size == exp["S_mec"] == oracle_mod.S_mec(d)
    cpo = oracle_mod.encode(d, x, cps=False)
    cps = oracle_mod.encode(d, x, cps=True)
    n_cpo = cpo["ptr"].size + cpo["da"].size + cpo["inn"].size
    n_cps = cps["ptr"].size + cps["da"].size + cps["inn"].size
    assert (n_cpo, n_cps) == (37, 36)
    # ptr length 17 = NOP 3 + 3 blocks of 6 - one NPF discount of (O_w - 1) (SI Eq. 3)
    assert oracle_mod.ptr_size_eq3(d, np.array([10 / 64]), count_npf=1) == 17


def test_fig1_pattern_helpers(oracle_mod):
    # pattern 14 (1110) -> 3 NZEs; 7 -> 7+K_w = 11 -> 7+2K_w = 15
    assert oracle_mod.pattern_size(14) == 2
    assert oracle_mod.next_offset(14, 1) == 1 and oracle_mod.next_offset(14, 2) == 1
    assert oracle_mod.pattern_size(15) == 3
    assert oracle_mod.next_offset(11, 2) == 2        # 1011: bits 0,1,3
    assert oracle_mod.next_offset(13, 1) == 2        # 1101: bits 0,2,3


def test_fig1_conv_equals_direct_exactly(oracle_mod):
    d, x, _ = load_fig1()
    w = np.arange(1, 17, dtype=np.float32).reshape(1, 1, 4, 4) - 8.0
    ref = oracle_mod.direct_conv(d, x, w)
    for cps in (False, True):
        enc = oracle_mod.encode(d, x, cps=cps)
        got = oracle_mod.sparse_conv(d, enc, w)
        assert np.array_equal(got, ref)
    assert np.array_equal(oracle_mod.decode(d, oracle_mod.encode(d, x, cps=True)), x)


def test_fig1_first_nze_footprint(oracle_mod):
    """"the first NZE in overlap2 is 10 ... contributes to four output
    indices (i.e, O[0:1][0:1])"."""
    d, _, _ = load_fig1()
    x = np.zeros((1, 1, 8, 8), dtype=np.float32)
    x[0, 0, 1, 1] = 10.0
    w = np.ones((1, 1, 4, 4), dtype=np.float32)
    y = oracle_mod.sparse_conv(d, oracle_mod.encode(d, x), w)[0, 0]
    assert sorted(zip(*np.nonzero(y))) == [(0, 0), (0, 1), (1, 0), (1, 1)]
    assert oracle_mod.mac_count(d, x) == 4


def test_single_nze_mac_count(oracle_mod):
    """An NZE at (5, 3) of the 8x8 / 4x4 VALID frame: windows start at rows 2..4
    (3 of them) and columns 0..3 (4, it is an overlap4 column) -> 12 MACs."""
    d, _, _ = load_fig1()
    x = np.zeros((1, 1, 8, 8), dtype=np.float32)
    x[0, 0, 5, 3] = 1.0
    assert oracle_mod.mac_count(d, x) == 12


@pytest.mark.parametrize("bad", ["ptr", "in"])
def test_corrupt_streams_detected(oracle_mod, bad):
    d, x, _ = load_fig1()
    enc = oracle_mod.encode(d, x)
    if bad == "ptr":
        enc["ptr"][3] = 7          # wrong type tag
    else:
        enc["inn"] = enc["inn"][:-1]
    with pytest.raises(ValueError):
        oracle_mod.decode(d, enc)
