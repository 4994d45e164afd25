#!/usr/bin/env python
"""Generate csrc/dispatch_gen.cuh: the NZE-list replay loop of the register-tile
sparse conv as inline PTX, one specialisation per tile configuration.

Why generated PTX: NVVM lowers a C++ `switch` over the ~100 window positions into
a compare tree (~20 instructions per NZE); `brx.idx` over a `.branchtargets`
table gives one indexed branch.  Each case body is the static sequence of
packed `fma.rn.f32x2` (FFMA2, sm_100) that the NZE at that window position
contributes: acc[(k, k+32)][y][x] += v * W[(k, k+32)][l][m] for every tap
(l, m) whose output (y, x) lies in the tile and on the stride grid.

  python tools/gen_dispatch.py   (run by paper_2104_08314_b200/build.py)
"""
from __future__ import annotations

import os

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "..", "paper_2104_08314_b200", "csrc", "dispatch_gen.cuh")

# (R, S, SH, SW, TY, TX, KPL) -- must match the TileCfg instantiations in sparse_conv.cu
CONFIGS = [
    (3, 3, 1, 1, 8, 4, 2),
    (3, 3, 1, 1, 8, 4, 1),
    (3, 3, 1, 1, 4, 4, 4),
    (3, 3, 1, 1, 8, 4, 4),
    (3, 3, 2, 2, 4, 4, 2),
    (3, 3, 2, 2, 4, 4, 4),
    (1, 7, 1, 1, 8, 4, 2),
    (7, 1, 1, 1, 8, 4, 2),
]


def gen(R, S, SH, SW, TY, TX, KPL):
    WH, WW = (TY - 1) * SH + R, (TX - 1) * SW + S
    NP = KPL // 2 if KPL % 2 == 0 else KPL       # accumulator words per position
    packed = KPL % 2 == 0
    nacc = NP * TY * TX
    nw = NP * R * S

    def acc(p, y, x):
        return p * TY * TX + y * TX + x

    def wop(p, l, m):
        return nacc + p * R * S + l * S + m

    o_list = nacc + nw
    lines = []
    a = lines.append
    a("{")
    # Two register sets A / B hold consecutive list entries; the case bodies
    # exist twice (tables A and B).  A body of set X runs the FFMA2s with X's
    # value, then reloads X with the entry two positions ahead and dispatches
    # on the other set's case, which was loaded one full body earlier -- the
    # shared-memory and jump-table latencies overlap the FFMA2s and no register
    # rotation is needed.  Entries are 16 bytes {v, v, case, 0}: the value pair
    # is one 64-bit register (FFMA2 operand); the list ends with a sentinel
    # (case NCASE -> $Ldone) followed by one padding entry.
    a(".reg .b32 %%spcP, %%spcAC, %%spcBC;")
    a(".reg .b64 %%spcAV, %%spcBV, %%spcAX, %%spcBX;")
    if not packed:
        a(".reg .b32 %%spcAF, %%spcBF, %%spcAH, %%spcBH;")
    a(f"mov.b32 %%spcP, %{o_list};")
    a("ld.shared.v2.b64 {%%spcAV, %%spcAX}, [%%spcP];")
    a("ld.shared.v2.b64 {%%spcBV, %%spcBX}, [%%spcP+16];")
    a("add.u32 %%spcP, %%spcP, 32;")
    ncase = WH * WW
    for X, Y in (("A", "B"), ("B", "A")):
        a(f"$Ltab{X}%=: .branchtargets " + ", ".join(f"$L{X}{c}%=" for c in range(ncase)) + ", $Ldone%=;")
    a("cvt.u32.u64 %%spcAC, %%spcAX;")
    a("brx.idx.uni %%spcAC, $LtabA%=;")
    for X, Y in (("A", "B"), ("B", "A")):
        for c in range(ncase):
            hr, wr = divmod(c, WW)
            a(f"$L{X}{c}%=:")
            a(f"cvt.u32.u64 %%spc{Y}C, %%spc{Y}X;")
            if not packed:
                a(f"mov.b64 {{%%spc{X}F, %%spc{X}H}}, %%spc{X}V;")
            for l in range(R):
                for m in range(S):
                    y1, x1 = hr - l, wr - m
                    if y1 < 0 or x1 < 0 or y1 % SH or x1 % SW or y1 // SH >= TY or x1 // SW >= TX:
                        continue
                    y, x = y1 // SH, x1 // SW
                    for p in range(NP):
                        ai, wi = acc(p, y, x), wop(p, l, m)
                        if packed:
                            a(f"fma.rn.f32x2 %{ai}, %%spc{X}V, %{wi}, %{ai};")
                        else:
                            a(f"fma.rn.f32 %{ai}, %%spc{X}F, %{wi}, %{ai};")
            a(f"ld.shared.v2.b64 {{%%spc{X}V, %%spc{X}X}}, [%%spcP];")
            a("add.u32 %%spcP, %%spcP, 16;")
            a(f"brx.idx.uni %%spc{Y}C, $Ltab{Y}%=;")
    a("$Ldone%=:")
    a("}")
    asm = "\n".join('        "' + ln + '\\n"' for ln in lines)
    T = "unsigned long long" if packed else "float"
    cons_a = "l" if packed else "f"
    outs = ", ".join(f'"+{cons_a}"(acc[{p}][{y}][{x}])' for p in range(NP) for y in range(TY) for x in range(TX))
    ins = ", ".join(f'"{cons_a}"(w[{p}][{l}][{m}])' for p in range(NP) for l in range(R) for m in range(S))
    name = f"replay_{R}x{S}_s{SH}{SW}_t{TY}x{TX}_k{KPL}"
    return f"""
// R={R} S={S} stride=({SH},{SW}) tile {TY}x{TX}, {KPL} output channel(s) per lane; {ncase} window positions
__device__ __forceinline__ void {name}(unsigned list_smem, {T} (&acc)[{NP}][{TY}][{TX}],
                                       const {T} (&w)[{NP}][{R}][{S}]) {{
    asm volatile(
{asm}
        : {outs}
        : {ins}, "r"(list_smem));
}}
template <> struct Replay<{R}, {S}, {SH}, {SW}, {TY}, {TX}, {KPL}> {{
    static constexpr bool kPacked = {str(packed).lower()};
    using Word = {T};
    static constexpr int kSentinel = {ncase};  // lists: entries, sentinel, 1 padding entry
    __device__ __forceinline__ static void run(unsigned list_smem, {T} (&acc)[{NP}][{TY}][{TX}],
                                               const {T} (&w)[{NP}][{R}][{S}]) {{
        {name}(list_smem, acc, w);
    }}
}};
"""


def main():
    parts = ["// dispatch_gen.cuh -- GENERATED by tools/gen_dispatch.py; do not edit.",
             "// NZE-list replay loops (brx.idx jump table + FFMA2 case bodies) per tile config.",
             "#pragma once", "", "namespace spc {",
             "template <int R, int S, int SH, int SW, int TY, int TX, int KPL> struct Replay;"]
    for cfg in CONFIGS:
        parts.append(gen(*cfg))
    parts.append("}  // namespace spc\n")
    src = "\n".join(parts)
    if not os.path.exists(OUT) or open(OUT).read() != src:
        with open(OUT, "w") as f:
            f.write(src)
    print(OUT)


if __name__ == "__main__":
    main()
