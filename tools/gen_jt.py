"""Generate paper_1911_10175_b200/csrc/jt_blocks.cuh: jump-table FMA blocks.

For one tile configuration of tile_conv_kernel (FWD or BWI, KK output
channels per lane, TH x TW output tile per warp, R x S filter, stride STR)
every region pixel p has a static list of (output pixel, filter tap) pairs it
feeds.  In sparse mode only the NONZERO pixels of a channel are visited: a
chained dispatch (`brev`+`clz` finds the lowest set mask bit, `shfl` fetches
that pixel's value from the lane that loaded it, `brx.idx` jumps straight to
the pixel's FMA block) costs ~7 instructions and one indirect branch per
nonzero pixel and nothing per zero pixel -- the GPU form of the paper's
popcount/trailing-zero loop (P/include/spconv/vec.hpp:43-75).  The next
nonzero's index and value are computed before the current block's FMAs so
their latency overlaps the arithmetic.

The accumulators and filter taps stay C++ register arrays; each 32-pixel
word is one inline-PTX statement whose operands are those registers, so the
kernel code around it (staging, masks, epilogue) is ordinary CUDA C++.

Run:  python tools/gen_jt.py   (rewrites the header; `make` rebuilds).
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_1911_10175_b200", "csrc", "jt_blocks.cuh")
F32X2 = "--f32x2" in sys.argv

# BWW: (CHECK_INPUT, KK, TH, TW, R, S, STR) -- per (checked channel, word)
BWW_CONFIGS = [
    (True, 4, 4, 4, 3, 3, 1), (True, 2, 4, 4, 3, 3, 1),
    (False, 4, 2, 4, 3, 3, 1), (False, 2, 4, 4, 3, 3, 1),
]

# (FWD, KK, TH, TW, R, S, STR)
CONFIGS = [
    (True, 2, 4, 8, 3, 3, 1), (False, 2, 4, 8, 3, 3, 1),
    (True, 4, 4, 4, 3, 3, 1), (False, 4, 4, 4, 3, 3, 1),
    (True, 4, 4, 8, 3, 3, 1), (False, 4, 4, 8, 3, 3, 1),
    (True, 4, 7, 4, 3, 3, 1), (False, 4, 7, 4, 3, 3, 1),
    (True, 4, 4, 7, 3, 3, 1), (False, 4, 4, 7, 3, 3, 1),
]


def fdiv(a, b):
    return a // b


class Axis:
    def __init__(self, fwd, T, F, STR):
        self.fwd, self.T, self.F, self.STR = fwd, T, F, STR
        self.PAD = (F - 1) // 2
        self.R0 = 0 if fwd else fdiv(self.PAD - (F - 1), STR)
        self.EXT = (T - 1) * STR + F if fwd else fdiv(T - 1 + self.PAD, STR) - self.R0 + 1

    def target(self, r, f):  # mirrors Axis<>::target in tile_conv.cu
        if self.fwd:
            num = r - f
            if num < 0 or num % self.STR:
                return -1
            t = num // self.STR
            return t if t < self.T else -1
        t = (self.R0 + r) * self.STR + f - self.PAD
        return t if 0 <= t < self.T else -1


# Two-ahead dispatch: on entry to a pixel block the NEXT nonzero's index jn is
# already known, so the jump-table load for the block's own brx (ptxas lowers
# brx.idx to LDC + BRX) and the shfl of the next value issue at the top of the
# block and overlap its FMAs; the block itself finds the next-next index.
def dispatch_init(V):
    return ["brev.b32 jt, jm;", "clz.b32 jp, jt;", "sub.u32 jt, jm, 1;", "and.b32 jm, jm, jt;",
            "brev.b32 jt, jm;", "clz.b32 jn, jt;", "sub.u32 jt, jm, 1;", "and.b32 jm, jm, jt;",
            f"shfl.sync.idx.b32 jd, %{V}, jp, 31, -1;"]


def dispatch_block_head(V):
    return [f"shfl.sync.idx.b32 jdn, %{V}, jn, 31, -1;",
            "brev.b32 jt, jm;", "clz.b32 jq, jt;", "sub.u32 jt, jm, 1;", "and.b32 jm, jm, jt;"]


DISPATCH_TAIL = ["mov.f32 jd, jdn;", "mov.b32 jp, jn;", "mov.b32 jn, jq;", "brx.idx.uni jp, Ljt;"]


def word_asm(cfg, w):
    fwd, KK, TH, TW, R, S, STR = cfg
    ay, ax = Axis(fwd, TH, S, STR), Axis(fwd, TW, R, STR)
    RH, RWW = ay.EXT, ax.EXT
    RHW = RH * RWW
    NACC = TH * TW * KK
    TAPS = R * S
    gi = lambda f, j: NACC + f * KK + j
    V = NACC + TAPS * KK
    M = V + 1
    # packed f32x2 FMAs: accumulator and tap channel pairs live in .b64
    # registers (ptxas coalesces the packing movs away) and the pixel value is
    # broadcast to both halves (the FFMA2 scalar-operand form)
    # Off: measured 20-35% SLOWER on B200 -- inside the multi-block asm ptxas
    # does not coalesce the .b64 pairs with the C++ accumulators and emits a
    # MOV pair after every FFMA2 (tools/gen_jt.py --f32x2 to regenerate).
    P2 = F32X2 and KK % 2 == 0
    pk = []
    if P2:
        pk = [f".reg .b64 A<{NACC // 2}>, G<{TAPS * KK // 2}>, jdd;"]
        pk += [f"mov.b64 A{a // 2}, {{%{a}, %{a + 1}}};" for a in range(0, NACC, 2)]
        pk += [f"mov.b64 G{(i - NACC) // 2}, {{%{i}, %{i + 1}}};" for i in range(NACC, NACC + TAPS * KK, 2)]
    lines = ["{",
             ".reg .b32 jm, jt, jp, jn, jq;",
             ".reg .f32 jd, jdn;"] + pk + [
             f"mov.b32 jm, %{M};"] + dispatch_init(V) + [
             "Ljt: .branchtargets " + ", ".join(f"Lb{i}" for i in range(32)) + ", Lend;",
             "brx.idx.uni jp, Ljt;"]
    for i in range(32):
        p = 32 * w + i
        lines.append(f"Lb{i}:")
        if p >= RHW:
            lines.append("bra.uni Lend;")
            continue
        ry, rx = divmod(p, RWW)
        lines += dispatch_block_head(V)
        if P2:
            lines.append("mov.b64 jdd, {jd, jd};")
        for v in range(S):
            ty = ay.target(ry, v)
            if ty < 0:
                continue
            for u in range(R):
                tx = ax.target(rx, u)
                if tx < 0:
                    continue
                t = ty * TW + tx
                if P2:
                    for j in range(0, KK, 2):
                        a = t * KK + j
                        lines.append(f"fma.rn.f32x2 A{a // 2}, jdd, G{(gi(v * R + u, j) - NACC) // 2}, A{a // 2};")
                    continue
                for j in range(KK):
                    a = t * KK + j
                    lines.append(f"fma.rn.f32 %{a}, jd, %{gi(v * R + u, j)}, %{a};")
        lines += DISPATCH_TAIL
    lines += ["Lend:"]
    if P2:
        lines += [f"mov.b64 {{%{a}, %{a + 1}}}, A{a // 2};" for a in range(0, NACC, 2)]
    lines += ["}"]
    body = "\\n\\t".join(lines)
    outs = ", ".join(f'"+f"(acc[{t}][{j}])' for t in range(TH * TW) for j in range(KK))
    ins = ", ".join(f'"f"(g[{f}].v[{j}])' for f in range(TAPS) for j in range(KK)) + ', "f"(v), "r"(m)'
    return f'    asm volatile("{body}"\n                 : {outs}\n                 : {ins});'


def word_asm_pair(cfg, w):
    """word_asm with packed f32x2 FMAs on 64-bit operands: the accumulators
    and taps are passed as .b64 registers holding two fp32 channels each (the
    kernel keeps them in that form for the whole pass), so ptxas needs no
    packing moves; the pixel value is broadcast with mov.b64 {jd, jd}, which
    ptxas folds into the FFMA2 scalar-operand form."""
    fwd, KK, TH, TW, R, S, STR = cfg
    ay, ax = Axis(fwd, TH, S, STR), Axis(fwd, TW, R, STR)
    RH, RWW = ay.EXT, ax.EXT
    RHW = RH * RWW
    KP = KK // 2
    NACC = TH * TW * KP
    TAPS = R * S
    gi = lambda f, j: NACC + f * KP + j
    V = NACC + TAPS * KP
    M = V + 1
    lines = ["{",
             ".reg .b32 jm, jt, jp, jn, jq;",
             ".reg .f32 jd, jdn;",
             ".reg .b64 jdd;",
             f"mov.b32 jm, %{M};"] + dispatch_init(V) + [
             "Ljt: .branchtargets " + ", ".join(f"Lb{i}" for i in range(32)) + ", Lend;",
             "brx.idx.uni jp, Ljt;"]
    for i in range(32):
        p = 32 * w + i
        lines.append(f"Lb{i}:")
        if p >= RHW:
            lines.append("bra.uni Lend;")
            continue
        ry, rx = divmod(p, RWW)
        lines += ["mov.b64 jdd, {jd, jd};"] + dispatch_block_head(V)
        for v in range(S):
            ty = ay.target(ry, v)
            if ty < 0:
                continue
            for u in range(R):
                tx = ax.target(rx, u)
                if tx < 0:
                    continue
                t = ty * TW + tx
                for j in range(KP):
                    a = t * KP + j
                    lines.append(f"fma.rn.f32x2 %{a}, jdd, %{gi(v * R + u, j)}, %{a};")
        lines += DISPATCH_TAIL
    lines += ["Lend:", "}"]
    body = "\\n\\t".join(lines)
    outs = ", ".join(f'"+l"(acc[{t}][{j}])' for t in range(TH * TW) for j in range(KP))
    ins = ", ".join(f'"l"(g[{f}].p[{j}])' for f in range(TAPS) for j in range(KP)) + ', "f"(v), "r"(m)'
    return f'    asm volatile("{body}"\n                 : {outs}\n                 : {ins});'


def bww_word_asm(cfg, w):
    """acc[tap][j] += d * O[q][j] for every (tap, other-tile pixel q) a checked
    pixel feeds (tile_bww.cu's in-line loop, restated as static lists)."""
    ci, KK, TH, TW, R, S, STR = cfg
    irh, irw = (TH - 1) * STR + S, (TW - 1) * STR + R
    crh, crw = (irh, irw) if ci else (TH, TW)
    otw = TW if ci else irw
    chw = crh * crw
    TAPS = R * S
    NACC = TAPS * KK
    NO = (TH * TW if ci else irh * irw)
    oi = lambda q, j: NACC + q * KK + j
    V = NACC + NO * KK
    M = V + 1
    lines = ["{", ".reg .b32 jm, jt, jp, jn;", ".reg .f32 jd, jdn;", f"mov.b32 jm, %{M};",
             "brev.b32 jt, jm;", "clz.b32 jp, jt;", "sub.u32 jt, jm, 1;", "and.b32 jm, jm, jt;",
             f"shfl.sync.idx.b32 jd, %{V}, jp, 31, -1;",
             "Ljt: .branchtargets " + ", ".join(f"Lb{i}" for i in range(32)) + ", Lend;",
             "brx.idx.uni jp, Ljt;"]
    for i in range(32):
        p = 32 * w + i
        lines.append(f"Lb{i}:")
        if p >= chw:
            lines.append("bra.uni Lend;")
            continue
        ry, rx = divmod(p, crw)
        lines += ["brev.b32 jt, jm;", "clz.b32 jn, jt;", "sub.u32 jt, jm, 1;", "and.b32 jm, jm, jt;",
                  f"shfl.sync.idx.b32 jdn, %{V}, jn, 31, -1;"]
        for v in range(S):
            for u in range(R):
                if ci:
                    ny, nx = ry - v, rx - u
                    if ny < 0 or nx < 0 or ny % STR or nx % STR or ny // STR >= TH or nx // STR >= TW:
                        continue
                    q = (ny // STR) * otw + nx // STR
                else:
                    q = (ry * STR + v) * otw + rx * STR + u
                for j in range(KK):
                    a = (v * R + u) * KK + j
                    lines.append(f"fma.rn.f32 %{a}, jd, %{oi(q, j)}, %{a};")
        lines += ["mov.f32 jd, jdn;", "brx.idx.uni jn, Ljt;"]
    lines += ["Lend:", "}"]
    body = "\\n\\t".join(lines)
    outs = ", ".join(f'"+f"(acc[{f}][{j}])' for f in range(TAPS) for j in range(KK))
    ins = ", ".join(f'"f"(O[{q}][{j}])' for q in range(NO) for j in range(KK)) + ', "f"(v), "r"(m)'
    return f'        asm volatile("{body}"\n                     : {outs}\n                     : {ins});'


def main():
    out = ["// GENERATED by tools/gen_jt.py -- do not edit.",
           "// Jump-table (brx.idx) FMA blocks for tile_conv_kernel's sparse mode; see the",
           "// generator's docstring.  One specialization per tile configuration.",
           "#pragma once", "", "namespace spc {", "",
           "template <bool FWD, int KK, int TH, int TW, int R, int S, int STR>",
           "struct JtBlocks {",
           "    static constexpr bool available = false;",
           "    template <int W>",
           "    struct Word {",
           "        template <class Acc, class Gv>",
           "        static __device__ __forceinline__ void run(Acc&, const Gv&, float, unsigned) {}",
           "    };",
           "};", ""]
    for cfg in CONFIGS:
        fwd, KK, TH, TW, R, S, STR = cfg
        RHW = Axis(fwd, TH, S, STR).EXT * Axis(fwd, TW, R, STR).EXT
        nword = (RHW + 31) // 32
        targs = f"{'true' if fwd else 'false'}, {KK}, {TH}, {TW}, {R}, {S}, {STR}"
        out += [f"template <>", f"struct JtBlocks<{targs}> {{",
                "    static constexpr bool available = true;",
                "    template <int W>",
                "    struct Word;",
                "};"]
        for w in range(nword):
            out += [f"template <>", f"struct JtBlocks<{targs}>::Word<{w}> {{",
                    "    template <class Acc, class Gv>",
                    "    static __device__ __forceinline__ void run(Acc& acc, const Gv& g, float v, unsigned m) {",
                    word_asm(cfg, w), "    }", "};", ""]
    out += ["// Pair form (KK % 4 == 0 configs): acc[t][KK/2] and tap vectors of .b64 lanes.",
            "template <bool FWD, int KK, int TH, int TW, int R, int S, int STR>",
            "struct JtBlocks2 {",
            "    static constexpr bool available = false;",
            "    template <int W>",
            "    struct Word {",
            "        template <class Acc, class Gv>",
            "        static __device__ __forceinline__ void run(Acc&, const Gv&, float, unsigned) {}",
            "    };",
            "};", ""]
    for cfg in CONFIGS:
        fwd, KK, TH, TW, R, S, STR = cfg
        if KK % 4:
            continue
        RHW = Axis(fwd, TH, S, STR).EXT * Axis(fwd, TW, R, STR).EXT
        targs = f"{'true' if fwd else 'false'}, {KK}, {TH}, {TW}, {R}, {S}, {STR}"
        out += ["template <>", f"struct JtBlocks2<{targs}> {{", "    static constexpr bool available = true;",
                "    template <int W>", "    struct Word;", "};"]
        for w in range((RHW + 31) // 32):
            out += ["template <>", f"struct JtBlocks2<{targs}>::Word<{w}> {{",
                    "    template <class Acc, class Gv>",
                    "    static __device__ __forceinline__ void run(Acc& acc, const Gv& g, float v, unsigned m) {",
                    word_asm_pair(cfg, w), "    }", "};", ""]
    out += ["template <bool CI, int KK, int TH, int TW, int R, int S, int STR>",
            "struct BwwJtBlocks {",
            "    static constexpr bool available = false;",
            "    template <int W>",
            "    struct Word {",
            "        template <class Acc, class Ov>",
            "        static __device__ __forceinline__ void run(Acc&, const Ov&, float, unsigned) {}",
            "    };",
            "};", ""]
    for cfg in BWW_CONFIGS:
        ci, KK, TH, TW, R, S, STR = cfg
        irh, irw = (TH - 1) * STR + S, (TW - 1) * STR + R
        chw = irh * irw if ci else TH * TW
        targs = f"{'true' if ci else 'false'}, {KK}, {TH}, {TW}, {R}, {S}, {STR}"
        out += ["template <>", f"struct BwwJtBlocks<{targs}> {{", "    static constexpr bool available = true;",
                "    template <int W>", "    struct Word;", "};"]
        for w in range((chw + 31) // 32):
            out += ["template <>", f"struct BwwJtBlocks<{targs}>::Word<{w}> {{",
                    "    template <class Acc, class Ov>",
                    "    static __device__ __forceinline__ void run(Acc& acc, const Ov& O, float v, unsigned m) {",
                    bww_word_asm(cfg, w), "    }", "};", ""]
    out += ["}  // namespace spc", ""]
    open(OUT, "w").write("\n".join(out))
    print("wrote", OUT, sum(len(x) for x in out), "bytes")


if __name__ == "__main__":
    main()
