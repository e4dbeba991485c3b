/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * "Modular SIMD arithmetic in MATHEMAGIX" (van der Hoeven, Lecerf, Quintin,
 * arXiv 1407.3383).  Citations are PAPER.md line numbers "P:n" with the
 * section / Function / Algorithm / Table they fall in.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1407_3383_b200/) never includes, links or calls it,
 * and this file includes nothing from the product path.
 *
 * Arithmetic primitives (the only ones used below):
 *   mulmod(a,b,p) = ((unsigned __int128)a*b) % p
 *   addmod(a,b,p) = ((unsigned __int128)a+b) % p
 *   submod(a,b,p) = ((unsigned __int128)a+p-b) % p
 *   powmod        = square-and-multiply over mulmod
 * Every "fast" method of the paper reaches exactly a result with a plain
 * definition; the oracle computes that definition (or a textbook algorithm
 * that is itself checked against the definition on small sizes in tests/).
 *
 * Parity pins: see tests/test_oracle.py (every exported function has at
 * least one pin that does not re-derive it from its own code).
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

#define EXPORT __attribute__((visibility("default")))

/* ---------------------------------------------------------------------- */
/* Scalar modular arithmetic: "Modulo p integers are stored as their */
/* representative in {0,...,p-1}"; Function 1 defines add.     */
/* ---------------------------------------------------------------------- */

EXPORT uint64_t or_addmod(uint64_t x, uint64_t y, uint64_t p) {
    /* (x + y) rem p, P:123 (Function 1 output). */
    return (uint64_t)(((u128)x + y) % p);
}

EXPORT uint64_t or_submod(uint64_t x, uint64_t y, uint64_t p) {
    /* (x - y) rem p; "Negation and subtraction ... in a similar manner". */
    return (uint64_t)(((u128)x + p - (y % p)) % p);
}

EXPORT uint64_t or_mulmod(uint64_t x, uint64_t y, uint64_t p) {
    /* (x y) rem p, the output of Functions 6/8/12. */
    return (uint64_t)(((u128)x * y) % p);
}

EXPORT uint64_t or_powmod(uint64_t b, uint64_t e, uint64_t p) {
    uint64_t r = 1 % p;
    b %= p;
    while (e) {
        if (e & 1) r = or_mulmod(r, b, p);
        b = or_mulmod(b, b, p);
        e >>= 1;
    }
    return r;
}

/* Deterministic primality for 64-bit integers: trial division by small
 * primes, then Miller-Rabin with the first 12 prime bases (exact for all
 * n < 3.3e24).  Used only to validate moduli ("p odd prime"). */
EXPORT int or_is_prime(uint64_t n) {
    static const uint64_t small[] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == small[i]) return 1;
        if (n % small[i] == 0) return 0;
    }
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        uint64_t x = or_powmod(small[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) {
            x = or_mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

/* 2-adic valuation of p - 1 (p = k 2^l + 1). */
EXPORT int or_two_adicity(uint64_t p) {
    uint64_t d = p - 1;
    int l = 0;
    if (d == 0) return 0;
    while ((d & 1) == 0) { d >>= 1; l++; }
    return l;
}

/* Multiplicative order of w modulo p when it divides 2^k: returns the least
 * j = 2^e with w^j = 1, or 0 if w^(2^k) != 1.  Definition of "primitive
 * n-th root of unity". */
EXPORT uint64_t or_order_pow2(uint64_t w, int k, uint64_t p) {
    uint64_t x = w % p;
    for (int e = 0; e <= k; e++) {
        if (x == 1) return (uint64_t)1 << e;
        x = or_mulmod(x, x, p);
    }
    return 0;
}

/* ---------------------------------------------------------------------- */
/* Precomputed constants of the reductions.                   */
/* ---------------------------------------------------------------------- */

/* r := ceil(log p / log 2), i.e. 2^(r-1) < p <= 2^r. */
EXPORT int or_bitsize_r(uint64_t p) {
    int r = 0;
    while (r < 64 && ((u128)1 << r) < p) r++;
    return r;
}

/* Table 3 profile parameters for Barrett's reduction.
 * profile: 2 => column "m <= n-2", 1 => "m <= n-1", 0 => "m <= n".
 * Outputs s, t, alpha_log2, h and q = floor(2^(s+t)/p). */
EXPORT int or_barrett_params(uint64_t p, int n, int profile,
                             int *r_out, int *s_out, int *t_out,
                             int *alpha_log2_out, int *h_out, uint64_t *q_out) {
    int r = or_bitsize_r(p);
    int s, t, a, h;
    if (p < 3) return -1;               /* MINUS2 breaks at p=2 */
    if (profile == 2) {                 /* m <= n-2 column */
        if (r > n - 2) return -2;
        s = r - 2 > 0 ? r - 2 : 0; t = n + 1; a = n - 2; h = 1;
    } else if (profile == 1) {          /* m <= n-1 column */
        if (r > n - 1) return -2;
        s = r - 1; t = n; a = n - 1; h = 2;
    } else {                            /* m <= n column */
        if (r > n) return -2;
        s = r - 1; t = n; a = n; h = 3;
    }
    *r_out = r; *s_out = s; *t_out = t; *alpha_log2_out = a; *h_out = h;
    *q_out = (uint64_t)((((u128)1) << (s + t)) / p);
    return 0;
}

/* Function 6 followed step by step, with its correction count
 * returned so tests can check Proposition 1's bound h.  a < alpha p.
 * Requires n <= 32 here so that L = u128 holds every intermediate. */
EXPORT uint64_t or_reduce_barrett_fn6(uint64_t a_lo, uint64_t a_hi, uint64_t p,
                                      int s, int t, uint64_t q, int *iters) {
    u128 a = ((u128)a_hi << 64) | a_lo;
    u128 b = a >> s;                    /* 1. L b = a >> s        */
    u128 c = (b * q) >> t;              /* 2. L c = (b * q) >> t  */
    u128 d = a - c * p;                 /* 3. L d = a - c * p     */
    int it = 0;
    while (d >= p) { d -= p; it++; }    /* 4. while (d >= p) ...  */
    if (iters) *iters = it;
    return (uint64_t)d;                 /* 5. return d            */
}

/* psi := floor(2^n y / p), the fixed-multiplicand pre-quotient of Function 8
 * (P:319).  With n = 32 this is Shoup's companion y' of the BASELINE. */
EXPORT uint64_t or_shoup_psi(uint64_t y, uint64_t p, int n) {
    return (uint64_t)((((u128)y) << n) / p);
}

/* Montgomery constants: 0 < chi < 2^m, 0 < rho < p,
 * rho 2^m - chi p = 1.  Computed from the definitions: rho = (2^m)^(-1) mod p
 * by Fermat (p prime) and chi = (rho 2^m - 1) / p. Also r2 = 2^(2m) mod p. */
EXPORT int or_montgomery_params(uint64_t p, int m, uint64_t *chi, uint64_t *rho,
                                uint64_t *r2) {
    if ((p & 1) == 0 || p < 3) return -1;
    uint64_t two_m = (uint64_t)((((u128)1) << m) % p);
    uint64_t rh = or_powmod(two_m, p - 2, p);
    u128 num = (((u128)rh) << m) - 1;
    if (num % p != 0) return -2;        /* p not prime: Fermat inverse wrong */
    *rho = rh;
    *chi = (uint64_t)(num / p);
    *r2 = or_mulmod(two_m, two_m, p);
    return 0;
}

/* Function 13 followed step by step, for m <= 63 (the u128
 * type plays L).  Returns (a rho) mod p for 0 <= a < 2^m p. */
EXPORT uint64_t or_reduce_montgomery_fn13(uint64_t a_lo, uint64_t a_hi, uint64_t p,
                                          int m, uint64_t chi) {
    u128 a = ((u128)a_hi << 64) | a_lo;
    u128 mu = (((u128)1) << m) - 1;
    u128 b = (a * chi) & mu;            /* 1. U b = (a * chi) & mu */
    u128 c = a + b * p;                 /* 2. L c = a + b * p      */
    u128 d = c >> m;                    /* 3. U d = c >> m         */
    return (uint64_t)((d >= p) ? d - p : d);   /* 5. (line 4 dead: no L overflow) */
}

/* ---------------------------------------------------------------------- */
/* Vector operations: the L2 "vector_linear" operations of P:797 on arrays. */
/* All inputs are uint64 arrays holding residues in [0, p).                */
/* ---------------------------------------------------------------------- */

EXPORT void or_vec_addmod(const uint64_t *x, const uint64_t *y, uint64_t *z,
                          size_t n, uint64_t p) {
    for (size_t i = 0; i < n; i++) z[i] = or_addmod(x[i], y[i], p);
}
EXPORT void or_vec_submod(const uint64_t *x, const uint64_t *y, uint64_t *z,
                          size_t n, uint64_t p) {
    for (size_t i = 0; i < n; i++) z[i] = or_submod(x[i], y[i], p);
}
EXPORT void or_vec_mulmod(const uint64_t *x, const uint64_t *y, uint64_t *z,
                          size_t n, uint64_t p) {
    for (size_t i = 0; i < n; i++) z[i] = or_mulmod(x[i], y[i], p);
}
/* Montgomery product: x y 2^(-m) mod p, i.e. REDC(x y). */
EXPORT void or_vec_montmul(const uint64_t *x, const uint64_t *y, uint64_t *z,
                           size_t n, uint64_t p, int m) {
    uint64_t rho = or_powmod((uint64_t)((((u128)1) << m) % p), p - 2, p);
    for (size_t i = 0; i < n; i++) z[i] = or_mulmod(or_mulmod(x[i], y[i], p), rho, p);
}
/* Montgomery representation x 2^m mod p. */
EXPORT void or_vec_to_mont(const uint64_t *x, uint64_t *z, size_t n, uint64_t p, int m) {
    uint64_t two_m = (uint64_t)((((u128)1) << m) % p);
    for (size_t i = 0; i < n; i++) z[i] = or_mulmod(x[i], two_m, p);
}
EXPORT void or_vec_shoup_psi(const uint64_t *y, uint64_t *z, size_t n, uint64_t p, int nbits) {
    for (size_t i = 0; i < n; i++) z[i] = or_shoup_psi(y[i], p, nbits);
}

/* ---------------------------------------------------------------------- */
/* Fourier transforms over Z/pZ, Section 5.1.                             */
/* ---------------------------------------------------------------------- */

/* [i]_k, the bitwise mirror of i in length k. */
EXPORT uint64_t or_bitrev(uint64_t i, int k) {
    uint64_t r = 0;
    for (int b = 0; b < k; b++)
        if (i & ((uint64_t)1 << b)) r |= (uint64_t)1 << (k - 1 - b);
    return r;
}

/* Primitive 2^k-th root from a generator g of (Z/pZ)^*: w = g^((p-1)/2^k). */
EXPORT uint64_t or_root_of_unity(uint64_t g, int k, uint64_t p) {
    return or_powmod(g, (p - 1) >> k, p);
}

/* FFT_w definition: out_i = sum_{j<n} w^(i j) a_j.  O(n^2). */
EXPORT void or_dft(const uint64_t *a, uint64_t *out, size_t n, uint64_t w, uint64_t p) {
    for (size_t i = 0; i < n; i++) {
        uint64_t wi = or_powmod(w, i, p);      /* w^i */
        uint64_t x = 1, acc = 0;               /* x = w^(i j) */
        for (size_t j = 0; j < n; j++) {
            acc = or_addmod(acc, or_mulmod(x, a[j], p), p);
            x = or_mulmod(x, wi, p);
        }
        out[i] = acc;
    }
}

/* One output of the definition: sum_j w^(i j) a_j.  O(n).
 * Used for sampled checks at sizes where the full O(n^2) sum is infeasible. */
EXPORT uint64_t or_dft_point(const uint64_t *a, size_t n, uint64_t w, uint64_t i, uint64_t p) {
    uint64_t wi = or_powmod(w, i % n, p);
    uint64_t x = 1, acc = 0;
    for (size_t j = 0; j < n; j++) {
        acc = or_addmod(acc, or_mulmod(x, a[j], p), p);
        x = or_mulmod(x, wi, p);
    }
    return acc;
}

/* Textbook iterative radix-2 NTT (Cooley-Tukey decimation in time):
 * bit-reversal copy, then log2 n levels of butterflies u +- w^j v.
 * Natural order in, natural order out; computes exactly FFT_w of P:889
 * (checked against or_dft for every n <= 2^12 in tests). In place. */
EXPORT void or_ntt(uint64_t *a, int k, uint64_t w, uint64_t p) {
    size_t n = (size_t)1 << k;
    for (size_t i = 0; i < n; i++) {
        size_t j = (size_t)or_bitrev(i, k);
        if (i < j) { uint64_t t = a[i]; a[i] = a[j]; a[j] = t; }
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        uint64_t wl = or_powmod(w, n / len, p);  /* primitive len-th root */
        for (size_t s = 0; s < n; s += len) {
            uint64_t x = 1;
            for (size_t j = 0; j < len / 2; j++) {
                uint64_t u = a[s + j];
                uint64_t v = or_mulmod(a[s + j + len / 2], x, p);
                a[s + j] = or_addmod(u, v, p);
                a[s + j + len / 2] = or_submod(u, v, p);
                x = or_mulmod(x, wl, p);
            }
        }
    }
}

/* Inverse transform: a_j = n^(-1) sum_i w^(-i j) ahat_i (reading of P:923,
 * "use the inverse of the TFFT"; R5 fixes the n^(-1) scaling). */
EXPORT void or_intt(uint64_t *a, int k, uint64_t w, uint64_t p) {
    size_t n = (size_t)1 << k;
    uint64_t winv = or_powmod(w, p - 2, p);
    or_ntt(a, k, winv, p);
    uint64_t ninv = or_powmod(n % p, p - 2, p);
    for (size_t i = 0; i < n; i++) a[i] = or_mulmod(a[i], ninv, p);
}

/* TFT order with l = n: position i holds ahat_{[i]_k}. */
EXPORT void or_to_bitrev(const uint64_t *in, uint64_t *out, int k) {
    size_t n = (size_t)1 << k;
    for (size_t i = 0; i < n; i++) out[i] = in[or_bitrev(i, k)];
}

/* Algorithm 1 with l = n, followed step by step, used only to
 * pin the four-step index maps (Proposition 15).  Output is
 * A(w^{[i]_k}) at position i.  n1 = 2^k1, n2 = n / n1. */
EXPORT void or_algorithm1(const uint64_t *a, uint64_t *out, int k, int k1,
                          uint64_t w, uint64_t p) {
    size_t n = (size_t)1 << k, n1 = (size_t)1 << k1;
    int k2 = k - k1;
    size_t n2 = n >> k1;
    uint64_t *bhat = (uint64_t *)malloc(n * sizeof(uint64_t));
    uint64_t *col = (uint64_t *)malloc(n2 * sizeof(uint64_t));
    uint64_t *row = (uint64_t *)malloc(n1 * sizeof(uint64_t));
    /* Step 1: b_{j2} = (a_{j2 n1}, ..., a_{(j2+1) n1 - 1}); TFFT over K^{n1}
     * of size n2 with root w^{n1}: for each lane j1, transform along j2 and
     * store in bit-mirrored order: bhat[i2][j1] = \hat b_{[i2]_{k2}, j1}. */
    uint64_t w1 = or_powmod(w, n1, p);
    for (size_t j1 = 0; j1 < n1; j1++) {
        for (size_t j2 = 0; j2 < n2; j2++) col[j2] = a[j2 * n1 + j1];
        or_ntt(col, k2, w1, p);
        for (size_t i2 = 0; i2 < n2; i2++)
            bhat[i2 * n1 + j1] = col[or_bitrev(i2, k2)];
    }
    /* Step 2: c_{j1}[i2] = \hat b_{[i2], j1} w^{j1 [i2]_{k2}}. */
    for (size_t i2 = 0; i2 < n2; i2++)
        for (size_t j1 = 0; j1 < n1; j1++)
            bhat[i2 * n1 + j1] = or_mulmod(bhat[i2 * n1 + j1],
                                           or_powmod(w, (uint64_t)j1 * or_bitrev(i2, k2), p), p);
    /* Step 3: TFFT over K^{lambda} of size n1 with root w^{n2}: for each i2,
     * transform along j1, bit-mirrored output. Step 4: position i2 n1 + i1
     * holds \hat c_{[i1]_{k1}, i2}. */
    uint64_t w2 = or_powmod(w, n2, p);
    for (size_t i2 = 0; i2 < n2; i2++) {
        for (size_t j1 = 0; j1 < n1; j1++) row[j1] = bhat[i2 * n1 + j1];
        or_ntt(row, k1, w2, p);
        for (size_t i1 = 0; i1 < n1; i1++)
            out[i2 * n1 + i1] = row[or_bitrev(i1, k1)];
    }
    free(bhat); free(col); free(row);
}

/* ---------------------------------------------------------------------- */
/* Section 5.2: polynomial product over Z/pZ.                             */
/* ---------------------------------------------------------------------- */

/* Schoolbook definition: c_k = sum_{i+j=k} a_i b_j mod p, k < la+lb-1. */
EXPORT void or_poly_mul_schoolbook(const uint64_t *a, size_t la, const uint64_t *b,
                                   size_t lb, uint64_t *c, uint64_t p) {
    if (la == 0 || lb == 0) return;
    size_t lc = la + lb - 1;
    for (size_t k = 0; k < lc; k++) c[k] = 0;
    for (size_t i = 0; i < la; i++)
        for (size_t j = 0; j < lb; j++)
            c[i + j] = or_addmod(c[i + j], or_mulmod(a[i], b[j], p), p);
}

/* TFT product of P:952: pad to n = 2^ceil(log2(la+lb-1)) (DESIGN R6), two
 * direct transforms, entry-wise product, one inverse transform.  Uses the
 * textbook or_ntt (itself pinned to the definition). w = g^((p-1)/n). */
EXPORT int or_poly_mul_ntt(const uint64_t *a, size_t la, const uint64_t *b, size_t lb,
                           uint64_t *c, uint64_t p, uint64_t g) {
    if (la == 0 || lb == 0) return 0;
    size_t lc = la + lb - 1;
    int k = 0;
    while (((size_t)1 << k) < lc) k++;
    if (k > or_two_adicity(p)) return -1;
    size_t n = (size_t)1 << k;
    uint64_t *fa = (uint64_t *)calloc(n, sizeof(uint64_t));
    uint64_t *fb = (uint64_t *)calloc(n, sizeof(uint64_t));
    memcpy(fa, a, la * sizeof(uint64_t));
    memcpy(fb, b, lb * sizeof(uint64_t));
    uint64_t w = or_root_of_unity(g, k, p);
    or_ntt(fa, k, w, p);
    or_ntt(fb, k, w, p);
    for (size_t i = 0; i < n; i++) fa[i] = or_mulmod(fa[i], fb[i], p);
    or_intt(fa, k, w, p);
    memcpy(c, fa, lc * sizeof(uint64_t));
    free(fa); free(fb);
    return 0;
}

/* Evaluate A(x) = sum a_i x^i mod p (Horner).  For the Schwartz-Zippel
 * check c(r) = a(r) b(r) of SURVEY 8(c) O6. */
EXPORT uint64_t or_poly_eval(const uint64_t *a, size_t la, uint64_t x, uint64_t p) {
    uint64_t acc = 0;
    for (size_t i = la; i-- > 0;) acc = or_addmod(or_mulmod(acc, x, p), a[i], p);
    return acc;
}

/* ---------------------------------------------------------------------- */
/* Section 5.3: integer product on little-endian 16-bit limbs.            */
/* ---------------------------------------------------------------------- */

/* Carry propagation = evaluation at 2^h with h = 16 ("A(2^h) = a"):
 * limbs_out = base-2^16 digits of sum_k coef[k] 2^(16 k), nout digits. */
EXPORT void or_carry_u16(const uint64_t *coef, size_t ncoef, uint16_t *out, size_t nout) {
    u128 acc = 0;
    for (size_t k = 0; k < nout; k++) {
        if (k < ncoef) acc += coef[k];
        out[k] = (uint16_t)(acc & 0xFFFF);
        acc >>= 16;
    }
}

/* Schoolbook integer product: c = a b exactly, na + nb output limbs. */
EXPORT void or_int_mul_schoolbook_u16(const uint16_t *a, size_t na, const uint16_t *b,
                                      size_t nb, uint16_t *c) {
    size_t nc = na + nb;
    for (size_t k = 0; k < nc; k++) c[k] = 0;
    for (size_t i = 0; i < na; i++) {
        uint64_t carry = 0;
        for (size_t j = 0; j < nb; j++) {
            uint64_t t = (uint64_t)a[i] * b[j] + c[i + j] + carry;
            c[i + j] = (uint16_t)(t & 0xFFFF);
            carry = t >> 16;
        }
        size_t k = i + nb;
        while (carry) {
            uint64_t t = (uint64_t)c[k] + carry;
            c[k] = (uint16_t)(t & 0xFFFF);
            carry = t >> 16;
            k++;
        }
    }
}

/* Kronecker segmentation product with one prime p (DESIGN R7):
 * chunks of h = 16 bits -> coefficient polynomials A, B with A(2^16) = a,
 * product C = A B by or_poly_mul_ntt over p (exact because every coefficient
 * is < min(na,nb) (2^16-1)^2 < p), then evaluation at 2^16 by carries.
 * Returns -1 if the coefficient bound or the 2-adicity is exceeded. */
EXPORT int or_int_mul_ntt_u16(const uint16_t *a, size_t na, const uint16_t *b, size_t nb,
                              uint16_t *c, uint64_t p, uint64_t g) {
    size_t nc = na + nb;
    if (na == 0 || nb == 0) { for (size_t k = 0; k < nc; k++) c[k] = 0; return 0; }
    size_t mn = na < nb ? na : nb;
    if ((u128)mn * 0xFFFE0001ull >= p) return -1;
    uint64_t *A = (uint64_t *)malloc(na * sizeof(uint64_t));
    uint64_t *B = (uint64_t *)malloc(nb * sizeof(uint64_t));
    uint64_t *C = (uint64_t *)malloc((na + nb - 1) * sizeof(uint64_t));
    for (size_t i = 0; i < na; i++) A[i] = a[i];
    for (size_t i = 0; i < nb; i++) B[i] = b[i];
    int rc = or_poly_mul_ntt(A, na, B, nb, C, p, g);
    if (rc == 0) or_carry_u16(C, na + nb - 1, c, nc);
    free(A); free(B); free(C);
    return rc;
}

/* a mod q for an integer given as 16-bit LE limbs (Horner at 2^16); used
 * for the "casting out primes" check (c mod q = (a mod q)(b mod q) mod q). */
EXPORT uint64_t or_limbs_mod(const uint16_t *a, size_t na, uint64_t q) {
    uint64_t acc = 0;
    for (size_t i = na; i-- > 0;) acc = or_addmod(or_mulmod(acc, 65536 % q, q), a[i] % q, q);
    return acc;
}
