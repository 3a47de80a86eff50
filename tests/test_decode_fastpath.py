"""The GPU decode fast path is exact: for qbits <= 25 and every q in
[-S, S], float32(float64(q)/S) == IEEE float32 q/S, and scaling by 2^e is
exact while the result stays normal (e in [-100, 127]).  The reference
computes float32(float64(q)/S * 2^e) (codec.py:168); the kernel uses
__fdiv_rn((float)q, (float)S) * 2^e on that range and the float64 formula
elsewhere (qbits 26, extreme exponents).  The cache-fill kernel computes the
same quotient as y0 = q * r, r = RN32(1/S), corrected once with two fmas
(y0 + fma(-y0, S, q) * r), also checked here for every q in [-S-1, S]."""

import os
import subprocess

import pytest

SRC = r"""
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <string.h>
static uint32_t bits(float f) { uint32_t u; memcpy(&u, &f, 4); return u; }
int main(void) {
    long bad = 0;
    for (int qb = 4; qb <= 25; qb++) {
        const long S = (1L << (qb - 1)) - 1;
        const float sf = (float)S;
        const float r = 1.0f / sf;
        for (long q = -S - 1; q <= S; q++) {
            const float ref = (float)((double)q / (double)S);
            const float fast = (float)q / sf;
            const float y0 = (float)q * r;
            const float mul = fmaf(fmaf(-y0, sf, (float)q), r, y0);
            if (bits(ref) != bits(fast) || bits(ref) != bits(mul)) bad++;
        }
    }
    /* scaling: float32(x * 2^e) == float32(x) * 2^e for normal results */
    uint64_t st = 88172645463325252ull;
    for (int e = -100; e <= 127; e++) {
        for (int t = 0; t < 20000; t++) {
            st ^= st << 13; st ^= st >> 7; st ^= st << 17;
            const int qb = 4 + (int)(st % 22);
            const long S = (1L << (qb - 1)) - 1;
            const long q = (long)((st >> 8) % (uint64_t)(2 * S + 1)) - S;
            const float ref = (float)((double)q / (double)S * ldexp(1.0, e));
            const float fast = ((float)q / (float)S) * ldexpf(1.0f, e);
            if (bits(ref) != bits(fast)) bad++;
        }
    }
    /* qbits 26 is NOT exact (documented fallback) */
    long bad26 = 0;
    const long S = (1L << 25) - 1;
    for (long q = -S; q <= S; q += 7) {
        if (bits((float)((double)q / (double)S)) != bits((float)q / (float)S)) bad26++;
    }
    printf("%ld %ld\n", bad, bad26);
    return 0;
}
"""


def test_fast_path_is_exhaustively_exact(tmp_path):
    c = tmp_path / "fp.c"
    exe = tmp_path / "fp"
    c.write_text(SRC)
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-o", str(exe), str(c), "-lm"], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=600).stdout.split()
    bad, bad26 = int(out[0]), int(out[1])
    assert bad == 0, f"{bad} mismatches on the fast-path domain"
    assert bad26 > 0, "qbits 26 unexpectedly exact (fallback would be unnecessary)"
