#!/usr/bin/env python3
"""Generates paper_2601_20174_b200/csrc/mt_jump_table.inc: jump polynomials of
MT19937-64 (the generator behind the reference's Rng, rng.hpp:22-71).

The state of MT19937-64 is a window of 312 words (x[p] .. x[p+311]) of the
linear recurrence

    x[i+312] = x[i+156] ^ ((x[i] & UM | x[i+1] & LM) >> 1) ^ (x[i+1] odd ? A : 0)

Let T move the window by one word. T is linear over GF(2) on the 19937 state
bits and its minimal polynomial phi has degree 19937, so for any J

    T^J = g_J(T),   g_J(x) = x^J mod phi(x) = sum_i g_i x^i,

and the window J words ahead is  XOR_{i : g_i = 1} window(p + i)  — the XOR of
the windows at the set coefficients (csrc/mt_jump.hpp does exactly that, on
the host and on the device).

This script finds phi by Berlekamp-Massey on one output bit of the generator,
computes g_J for J = 2^j, j = JMIN .. JMAX, by repeated squaring, checks the
small ones against plain stepping and writes them as 312-word bit sets.

Run:  python scripts/make_mt_jump_table.py [--check-only]
"""
import argparse
import os
import sys

NN, MM = 312, 156
MATRIX_A = 0xB5026F5AA96619E9
UM = 0xFFFFFFFF80000000
LM = 0x7FFFFFFF
MASK = (1 << 64) - 1
DEG = 19937
JMIN, JMAX = 17, 40  # jumps of 2^17 .. 2^40 words


def seed_state(seed):
    x = [seed & MASK]
    for i in range(1, NN):
        x.append((6364136223846793005 * (x[-1] ^ (x[-1] >> 62)) + i) & MASK)
    return x


def step(win):
    """window (list of 312 words) -> window one word ahead"""
    y = (win[0] & UM) | (win[1] & LM)
    new = win[MM] ^ (y >> 1) ^ (MATRIX_A if (win[1] & 1) else 0)
    return win[1:] + [new]


def stream(win, count):
    """x[p + 312 .. p + 312 + count) for the window at p (untempered)"""
    buf = list(win)
    for i in range(count):
        y = (buf[i] & UM) | (buf[i + 1] & LM)
        buf.append(buf[i + MM] ^ (y >> 1) ^ (MATRIX_A if (buf[i + 1] & 1) else 0))
    return buf


def temper(x):
    x ^= (x >> 29) & 0x5555555555555555
    x ^= (x << 17) & 0x71D67FFFEDA60000
    x ^= (x << 37) & 0xFFF7EEE000000000
    x ^= x >> 43
    return x & MASK


def berlekamp_massey(bits):
    """connection polynomial C (int, bit i = c_i, c_0 = 1) and its length L of the
    shortest LFSR with s[n] = sum_{i=1..L} c_i s[n-i] over GF(2)"""
    n_total = len(bits)
    # R: bit j = s[n_total - 1 - j], so (R >> (n_total - 1 - n)) has s[n - i] at bit i
    R = 0
    for b in bits:
        R = (R << 1) | b
    C, B, L, m = 1, 1, 0, 1
    for n in range(n_total):
        d = ((C & (R >> (n_total - 1 - n))).bit_count()) & 1
        if d == 0:
            m += 1
        elif 2 * L <= n:
            Tm = C
            C ^= B << m
            L = n + 1 - L
            B = Tm
            m = 1
        else:
            C ^= B << m
            m += 1
    return C, L


def poly_reverse(c, deg):
    out = 0
    for i in range(deg + 1):
        if (c >> i) & 1:
            out |= 1 << (deg - i)
    return out


def spread(p):
    """p(x)^2 over GF(2): bit i -> bit 2 i"""
    return int("0".join(bin(p)[2:]), 2)


def reduce(p, phi):
    for i in range(p.bit_length() - 1, DEG - 1, -1):
        if (p >> i) & 1:
            p ^= phi << (i - DEG)
    return p


def apply_jump(win, g):
    """window J ahead = XOR of the windows at the set coefficients of g_J"""
    xs = stream(win, DEG)  # x[p .. p + 312 + 19937)
    out = [0] * NN
    i = 0
    gg = g
    while gg:
        if gg & 1:
            for w in range(NN):
                out[w] ^= xs[i + w]
        gg >>= 1
        i += 1
    return out


def same_state(a, b):
    """windows agree on the 19937 state bits (the low 31 bits of word 0 are unused)"""
    return (a[0] & UM) == (b[0] & UM) and a[1:] == b[1:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--check-only", action="store_true")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(__file__), "..", "paper_2601_20174_b200", "csrc",
                                                  "mt_jump_table.inc"))
    args = ap.parse_args()

    # known answer: the 10000th output of a default-seeded std::mt19937_64
    xs = stream(seed_state(5489), 10000)
    assert temper(xs[NN + 9999]) == 9981545732273789042, "MT19937-64 restatement is wrong"

    # phi from 2 * 19937 + 64 output bits (bit 0 of the tempered output; any
    # nonzero linear functional of the state has minimal polynomial phi)
    nbits = 2 * DEG + 64
    xs = stream(seed_state(20174), nbits)
    bits = [temper(x) & 1 for x in xs[NN:NN + nbits]]
    C, L = berlekamp_massey(bits)
    assert L == DEG, L
    phi = poly_reverse(C, DEG)
    assert (phi >> DEG) == 1

    polys = {}
    p = 2  # x
    for j in range(1, JMAX + 1):
        p = reduce(spread(p), phi)
        polys[j] = p
    # checks against plain stepping: 2^10 and 2^13 words
    win = seed_state(7)
    for j in (10, 13):
        ref = stream(win, 1 << j)[(1 << j):(1 << j) + NN]
        assert same_state(apply_jump(win, polys[j]), ref), j
    # and composition: 2^17 = (2^13)^16 by 16 jumps of 2^13 vs one jump of 2^17
    w1 = win
    for _ in range(16):
        w1 = apply_jump(w1, polys[13])
    assert same_state(apply_jump(win, polys[17]), w1)
    print("phi degree", DEG, "weight", phi.bit_count(), "- jump polynomials verified", file=sys.stderr)
    if args.check_only:
        return

    with open(args.out, "w") as f:
        f.write("// Generated by scripts/make_mt_jump_table.py — do not edit.\n")
        f.write("// kMtJump[j - kMtJumpMinLog2]: coefficients of x^(2^j) mod phi(x) of MT19937-64,\n")
        f.write("// bit i of the 312-word set = coefficient of x^i (degree < 19937).\n")
        f.write("constexpr int kMtJumpMinLog2 = %d;\n" % JMIN)
        f.write("constexpr int kMtJumpMaxLog2 = %d;\n" % JMAX)
        f.write("static const unsigned long long kMtJump[%d][312] = {\n" % (JMAX - JMIN + 1))
        for j in range(JMIN, JMAX + 1):
            g = polys[j]
            words = [(g >> (64 * w)) & MASK for w in range(NN)]
            f.write("    {  // x^(2^%d)\n" % j)
            for r in range(0, NN, 4):
                f.write("        " + ", ".join("0x%016xull" % w for w in words[r:r + 4]) + ",\n")
            f.write("    },\n")
        f.write("};\n")
    print("wrote", os.path.normpath(args.out), file=sys.stderr)


if __name__ == "__main__":
    main()
