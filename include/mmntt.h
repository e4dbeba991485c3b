/*
 * mmntt.h -- C ABI of the B200-native hot path of
 *   J. van der Hoeven, G. Lecerf, G. Quintin, "Modular SIMD arithmetic in
 *   MATHEMAGIX" (arXiv 1407.3383).
 * Citations "P:n" are lines of the paper's text with the section,
 * Function, Algorithm or Table they fall in.
 *
 * Conventions (all entry points):
 *  - Pointers named x, y, z, a, b, c, in, out are DEVICE pointers owned by the
 *    caller (allocated e.g. by torch); the library only borrows them for the
 *    duration of the stream-ordered work it enqueues.
 *  - Every compute call is asynchronous on `stream` (a cudaStream_t, passed as
 *    void* so this header needs no CUDA include; NULL = legacy default
 *    stream).  Only the *_create / *_destroy / setup calls synchronise the
 *    device (and, under MMNTT_DEBUG=1, the range checks the stream).
 *    Temporaries and per-stream workspaces are stream-ordered allocations
 *    (cudaMallocAsync), so calls on different streams never share scratch.
 *  - Residues are canonical: inputs must lie in [0, p) ("stored as
 *    their representative in {0, ..., p-1}"), outputs always do.  Inputs are
 *    trusted unless the environment variable MMNTT_DEBUG=1 is set, in which
 *    case inputs are range-checked on the device and MM_E_RANGE is returned.
 *  - Calls never fall back to a slower path: unsupported moduli or sizes
 *    return a status.  mm_last_error() gives a thread-local message.
 *  - Contexts and plans are created and destroyed by the library (owned by
 *    it); they are immutable after creation and may be shared across streams.
 */
#ifndef MMNTT_H
#define MMNTT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MM_OK = 0,
    MM_E_INVALID_MODULUS = 1, /* p < 3, even, composite, or not k 2^l + 1 (NTT) */
    MM_E_PROFILE = 2,         /* p too wide for the requested variant (e.g. lazy NTT needs p < 2^30) */
    MM_E_UNSUPPORTED_SIZE = 3,/* 2^log2n does not divide p - 1, or log2n out of range */
    MM_E_BAD_ROOT = 4,        /* omega^(n/2) != p - 1: not a primitive 2^log2n-th root */
    MM_E_RANGE = 5,           /* debug check: an input residue >= p */
    MM_E_SIZE_OVERFLOW = 6,   /* int_mul coefficient bound min(na,nb)(2^16-1)^2 >= p, or length too large */
    MM_E_ALIAS = 7,           /* forbidden aliasing between input and output buffers */
    MM_E_CUDA = 8,            /* a CUDA runtime call failed (message in mm_last_error) */
    MM_E_NCCL = 9,            /* reserved for the distributed layer */
    MM_E_ARG = 10             /* null pointer / bad enum / bad size argument */
} mm_status;

typedef enum { MM_MUL_BARRETT = 0, MM_MUL_SHOUP = 1, MM_MUL_MONTGOMERY = 2 } mm_mul_variant;
typedef enum { MM_ORDER_NATURAL = 0, MM_ORDER_BITREV = 1 } mm_order;

typedef struct mm_mod32 mm_mod32;
typedef struct mm_mod64 mm_mod64;
typedef struct mm_modf64 mm_modf64;
typedef struct mm_ntt_plan mm_ntt_plan;

/* Thread-local description of the last non-OK status. */
const char *mm_last_error(void);
/* Library version string. */
const char *mm_version(void);

/* ------------------------------------------------------------------------
 * Modulus context.  Precomputes, on the host, for a 32-bit p:
 *   r (2^(r-1) < p <= 2^r); the Table-3 Barrett profile:
 *   m <= n-2 -> (s, t, h) = (max(r-2,0), n+1, 1), m <= n-1 -> (r-1, n, 2),
 *   m <= n -> (r-1, n, 3), with q = floor(2^(s+t)/p); the Montgomery
 *   constants for R = 2^32: p^-1 mod 2^32 and R^2 mod p.
 * p must be an odd prime >= 3 (Montgomery needs p odd).
 * Returns MM_E_INVALID_MODULUS otherwise.  *ctx is owned by the library. */
mm_status mm_mod32_create(uint32_t p, mm_mod32 **ctx);
void mm_mod32_destroy(mm_mod32 *ctx);
/* Read back the precomputed constants (for tests): out[0..7] =
 * {p, r, s, t, h, q, pinv (p^-1 mod 2^32), r2 (2^64 mod p)}. */
mm_status mm_mod32_info(const mm_mod32 *ctx, uint64_t out[8]);

/* ------------------------------------------------------------------------
 * Elementwise vector operations over n uint32 residues (the
 * "vector_linear" operations of P:797 with the modular kernels of S2).
 * z may alias x or y (in place); y_shoup may not alias z.
 *   mm_modadd_u32 : z_i = (x_i + y_i) rem p      (Function 1/2/4)
 *   mm_modsub_u32 : z_i = (x_i - y_i) rem p
 *   mm_modmul_u32 : BARRETT -> x_i y_i rem p     (Function 6 + Table 3)
 *                   SHOUP   -> x_i y_i rem p, needs y_shoup_i = floor(y_i 2^32 / p)
 *                              (Function 8); y_shoup ignored otherwise
 *                   MONTGOMERY -> x_i y_i 2^-32 rem p (Function 13 / REDC)
 *   mm_shoup_precompute_u32 : z_i = floor(y_i 2^32 / p)  (psi of P:319, n = 32)
 *   mm_to_mont_u32  : z_i = x_i 2^32 rem p        (Montgomery representation)
 *   mm_from_mont_u32: z_i = x_i 2^-32 rem p
 * Layout: contiguous arrays; 16-byte aligned pointers get 128-bit accesses,
 * others take a scalar path (same results). */
mm_status mm_modadd_u32(const mm_mod32 *ctx, const uint32_t *x, const uint32_t *y, uint32_t *z,
                        size_t n, void *stream);
mm_status mm_modsub_u32(const mm_mod32 *ctx, const uint32_t *x, const uint32_t *y, uint32_t *z,
                        size_t n, void *stream);
mm_status mm_modmul_u32(const mm_mod32 *ctx, mm_mul_variant v, const uint32_t *x, const uint32_t *y,
                        const uint32_t *y_shoup, uint32_t *z, size_t n, void *stream);
mm_status mm_shoup_precompute_u32(const mm_mod32 *ctx, const uint32_t *y, uint32_t *y_shoup, size_t n,
                                  void *stream);
mm_status mm_to_mont_u32(const mm_mod32 *ctx, const uint32_t *x, uint32_t *z, size_t n, void *stream);
mm_status mm_from_mont_u32(const mm_mod32 *ctx, const uint32_t *x, uint32_t *z, size_t n, void *stream);
/* The binary operations above on HOST vectors (x, y, y_shoup, z: n packed
 * uint32 residues in page-locked memory for overlap; z may alias x or y):
 * the vectors are cut into chunks that upload (own stream), run the device
 * operation (the caller's `stream`) and download (own stream) through three
 * library-owned device slots, so both PCIe directions overlap.  Same values
 * as mm_modadd_u32 / mm_modsub_u32 / mm_modmul_u32 of the variant; y_shoup
 * is read for MM_OP_MUL_SHOUP only (MM_E_ARG when null).  n = 0 is a no-op.
 * Asynchronous with respect to the host: `stream` is ordered after the last
 * download. */
typedef enum {
    MM_OP_ADD = 0, MM_OP_SUB = 1, MM_OP_MUL_BARRETT = 2, MM_OP_MUL_SHOUP = 3, MM_OP_MUL_MONTGOMERY = 4
} mm_host_op;
mm_status mm_modop_u32_host(const mm_mod32 *ctx, mm_host_op op, const uint32_t *x, const uint32_t *y,
                            const uint32_t *y_shoup, uint32_t *z, size_t n, void *stream);

/* ------------------------------------------------------------------------
 * 64-bit modulus context (SURVEY §8(b) mm_mod64_create; BASELINE C4 / C5's
 * p = 2^64 - 2^32 + 1, the only 64-bit modulus of this build, else
 * MM_E_INVALID_MODULUS).  The paper's 64-bit reductions are the generic
 * Barrett / Montgomery forms at m = n = 64; this modulus has the
 * special reduction 2^64 = 2^32 - 1, 2^96 = -1 (mod p) (R11).
 *   mm_modadd_u64 / mm_modsub_u64 / mm_modmul_u64 : z_i = (x_i op y_i) rem p
 * over n uint64 residues in [0, p) (canonical outputs), device pointers,
 * async on stream, in place allowed, MMNTT_DEBUG=1 range-checks the inputs. */
mm_status mm_mod64_create(uint64_t p, mm_mod64 **ctx);
void mm_mod64_destroy(mm_mod64 *ctx);
mm_status mm_modadd_u64(const mm_mod64 *ctx, const uint64_t *x, const uint64_t *y, uint64_t *z, size_t n,
                        void *stream);
mm_status mm_modsub_u64(const mm_mod64 *ctx, const uint64_t *x, const uint64_t *y, uint64_t *z, size_t n,
                        void *stream);
mm_status mm_modmul_u64(const mm_mod64 *ctx, const uint64_t *x, const uint64_t *y, uint64_t *z, size_t n,
                        void *stream);

/* ------------------------------------------------------------------------
 * Batched NTT plans.
 * FFT_w of length n = 2^log2n: out_i = sum_j w^(i j) in_j.
 *   word_bits = 32: p an odd prime < 2^30 (lazy butterflies in [0, 4p));
 *   word_bits = 64: p = 2^64 - 2^32 + 1 only.
 * omega must have exact order n: omega^(n/2) = p - 1 (else MM_E_BAD_ROOT);
 * 2^log2n must divide p - 1 (else MM_E_UNSUPPORTED_SIZE); 1 <= log2n <= 24
 * (32-bit) or 26 (64-bit).
 * `batch` independent transforms, rows contiguous with row stride n elements
 * (uint32 for 32-bit, uint64 for 64-bit).
 * Transforms of length <= 2^13 (2^12 for FP64 residues) run as one shared-memory pass per row;
 * longer ones use Algorithm 1 with l = n as a two-pass four-step
 * n = n2 x n1 (column pass + twiddle, row pass).
 * Creating a plan builds the twiddle tables on the device (one sync). */
/* word_bits selects the residue type: 32 (uint32_t, p < 2^30), 64 (uint64_t,
 * p = 2^64 - 2^32 + 1) or 52 (double holding integers in [0, p), odd prime
 * p < 2^50: Function 16 products and Function 17 sums on the FP64 pipe,
 * paper §3 / Table 12; four-step blocks and int_mul take 32 / 64 only). */
mm_status mm_ntt_plan_create(int word_bits, uint64_t p, int log2n, uint64_t omega, size_t batch,
                             mm_ntt_plan **plan);
void mm_ntt_plan_destroy(mm_ntt_plan *plan);
/* out[0..5] = {n1 (row length), n2 (column length), passes, 0 (plans hold no
 * workspace: NATURAL-order four-step calls permute through a stream-ordered
 * temporary), word_bits, batch} */
mm_status mm_ntt_plan_info(const mm_ntt_plan *plan, uint64_t out[6]);

/* Forward: in (natural order) -> out in `order`:
 *   MM_ORDER_NATURAL: out[i] = ahat_i;  MM_ORDER_BITREV: out[i] = ahat_{[i]_k},
 *   the TFT order of P:893 (what Algorithm 1 returns).
 * in == out (in place) is allowed. */
mm_status mm_ntt_forward(const mm_ntt_plan *plan, const void *in, void *out, mm_order order, void *stream);
/* Inverse: a_j = n^-1 sum_i w^(-i j) ahat_i (n^-1 included, R5),
 * `order` = order of the INPUT spectrum; output natural.  In place allowed. */
mm_status mm_ntt_inverse(const mm_ntt_plan *plan, const void *in, void *out, mm_order order, void *stream);

/* ------------------------------------------------------------------------
 * Polynomial product mod p: for each of `batch`
 * pairs, c[k] = sum_{i+j=k} a[i] b[j] mod p, 0 <= k < la + lb - 1.
 * a: [batch][la], b: [batch][lb], c: [batch][la+lb-1], rows contiguous.
 * Transform length n = 2^ceil(log2(la+lb-1)) (zero padding), root
 * w = g^((p-1)/n) for a generator g of (Z/pZ)^*.  Two forward transforms,
 * pointwise product with n^-1 folded in, one inverse.
 * c must not alias a or b (MM_E_ALIAS).  word_bits/p as for plans. */
mm_status mm_poly_mul(int word_bits, uint64_t p, uint64_t g, const void *a, size_t la, const void *b,
                      size_t lb, void *c, size_t batch, void *stream);
/* The same product with explicit row strides (leading dimensions, in
 * elements, BLAS-style): row r of a starts at a + r lda (lda >= la), of b at
 * b + r ldb, of c at c + r ldc (ldc >= la + lb - 1; elements of a c row beyond
 * la + lb - 1 are not written).  mm_poly_mul = lda = la, ldb = lb,
 * ldc = la + lb - 1.  A 128-byte multiple ldc keeps every output row
 * line-aligned (the packed layout with odd la + lb - 1 splits sectors between
 * neighbouring column tiles). */
/* The same product with HOST operands and result (a: [batch][la], b:
 * [batch][lb], c: [batch][la+lb-1], packed, page-locked memory for overlap):
 * the batch is cut into chunks that upload (own stream), multiply (the
 * caller's `stream`) and download (own stream) as a three-slot pipeline, so
 * the PCIe copies in both directions overlap the kernels.  Asynchronous with
 * respect to the host: `stream` is ordered after the last download (callers
 * synchronise it before reading c).  Device memory (3 chunk slots) is owned by
 * the library and reused. */
mm_status mm_poly_mul_host(int word_bits, uint64_t p, uint64_t g, const void *a, size_t la, const void *b,
                           size_t lb, void *c, size_t batch, void *stream);
mm_status mm_poly_mul_ld(int word_bits, uint64_t p, uint64_t g, const void *a, size_t la, size_t lda,
                         const void *b, size_t lb, size_t ldb, void *c, size_t ldc, size_t batch, void *stream);

/* FFT_w of P:887-893 (mm_ntt_forward / mm_ntt_inverse above) with HOST input
 * and output: in, out: [plan batch][2^log2n] elements, packed, page-locked
 * memory for overlap; in == out is allowed.  The batch rows are cut into
 * chunks that upload (own stream), transform (the caller's `stream`) and
 * download (own stream) through the three library-owned device slots of
 * mm_poly_mul_host, so both PCIe directions overlap the kernels; a plan of
 * batch 1 is one chunk (no overlap).  Same value and order semantics as the
 * device calls; asynchronous with respect to the host: `stream` is ordered
 * after the last download.  Errors: MM_E_ARG (null pointer, bad order),
 * MM_E_CUDA. */
mm_status mm_ntt_forward_host(const mm_ntt_plan *plan, const void *in, void *out, mm_order order, void *stream);
mm_status mm_ntt_inverse_host(const mm_ntt_plan *plan, const void *in, void *out, mm_order order, void *stream);

/* ------------------------------------------------------------------------
 * Modular vectors over IEEE doubles (paper §3; SURVEY §8(f)
 * item 3): residues of an odd p < 2^50 held as integral doubles in [0, p).
 *   mm_modf64_create : u = 1.0 / p rounded to nearest; p >= 2^50
 *       -> MM_E_PROFILE (Function 16 needs m <= l - 2 = 50).
 *   mm_modadd_f64 : Function 17, a = x + y, b = a - p, blend on
 *       the sign of b.       mm_modsub_f64 : the same for x - y (+ p).
 *   mm_modmul_f64 : Function 16 / 18: h = x y, l = fma(x, y, -h),
 *       c = floor(h u), e = fma(-c, p, h) + l, one correction each way
 *       (Proposition 13).
 * Device vectors, n elements, async on stream, in place allowed; outputs in
 * [0, p) for inputs in [0, p) (trusted precondition). */
mm_status mm_modf64_create(uint64_t p, mm_modf64 **ctx);
void mm_modf64_destroy(mm_modf64 *ctx);
mm_status mm_modadd_f64(const mm_modf64 *ctx, const double *x, const double *y, double *z, size_t n, void *stream);
mm_status mm_modsub_f64(const mm_modf64 *ctx, const double *x, const double *y, double *z, size_t n, void *stream);
mm_status mm_modmul_f64(const mm_modf64 *ctx, const double *x, const double *y, double *z, size_t n, void *stream);

/* ------------------------------------------------------------------------
 * Numeric reductions in float / double (paper §3.2-3.3; SURVEY
 * §8(f) item 3): residues of an odd p held as integral floats (fbits = 32,
 * trailing field l = 23) or doubles (fbits = 64, l = 52); m = bit size of p
 * (p < 2^m); u = 1.0 / p rounded to nearest, u-bar = 1.0 / p rounded
 * toward +inf.  The GPU rounds per instruction, so "the current
 * rounding mode" of the paper is the mode of every operation of the variant.
 *   MM_NUM_F14      Function 14, u, to nearest, both corrections;
 *                   m <= l/2 (double 26, float 11), inputs a < 2^(l/2) p.
 *   MM_NUM_F14_UP   Function 14 with u-bar, every operation toward +inf,
 *                   line 4 dropped (Proposition 10).
 *   MM_NUM_F15_UP   Function 15: u-bar, toward +inf, no correction
 *                   (Proposition 11); m <= (l-1)/2 (double 25, float 11),
 *                   inputs a < 2^floor((l-1)/2) p.
 *   MM_NUM_F15_NEAR Function 15 in round-to-nearest (Remark 12): only
 *                   for p prime and a = x y with x, y residues (mulmod only).
 *   MM_NUM_F16      Function 16, u, to nearest; m <= l - 2
 *                   (double 50, float 21) -- the product of mm_modmul_f64.
 *   MM_NUM_F16_UP   Function 16 with u-bar, toward +inf, line 7 dropped
 *                   (Proposition 13).
 * mm_modnum_create : p odd >= 3 with m <= l - 2 (else MM_E_INVALID_MODULUS /
 *     MM_E_PROFILE); a variant whose bound m exceeds returns MM_E_PROFILE at
 *     the call.  *ctx owned by the library.
 * mm_modnum_info   : out[0..5] = {p, u, u-bar, l, m, fbits}.
 * mm_mulmod_num    : z_i = (x_i y_i) rem p for residues x_i, y_i in [0, p)
 *     (F14 / F15 on the exact product a = x y, 2m <= l; F16 on the factors).
 * mm_reduce_num    : z_i = a_i rem p for integral a_i in [0, alpha p)
 *     (F14 / F14_UP / F15_UP only; MM_E_ARG for F16, MM_E_INVALID_MODULUS
 *     for F15_NEAR).
 * Device vectors of float (fbits 32) or double (64), n elements, async on
 * stream, in place allowed; 16-byte aligned vectors take 128-bit accesses.
 * Inputs are trusted unless MMNTT_DEBUG=1 (then out-of-domain inputs return
 * MM_E_RANGE; that check synchronises the stream). */
typedef enum {
    MM_NUM_F14 = 0,
    MM_NUM_F14_UP = 1,
    MM_NUM_F15_UP = 2,
    MM_NUM_F15_NEAR = 3,
    MM_NUM_F16 = 4,
    MM_NUM_F16_UP = 5
} mm_num_variant;
typedef struct mm_modnum mm_modnum;
mm_status mm_modnum_create(int fbits, uint64_t p, mm_modnum **ctx);
void mm_modnum_destroy(mm_modnum *ctx);
mm_status mm_modnum_info(const mm_modnum *ctx, double out[6]);
mm_status mm_mulmod_num(const mm_modnum *ctx, mm_num_variant v, const void *x, const void *y, void *z, size_t n,
                        void *stream);
mm_status mm_reduce_num(const mm_modnum *ctx, mm_num_variant v, const void *a, void *z, size_t n, void *stream);

/* Truncated product (Algorithm 1 with l < n):
 * the same c = a b mod p as mm_poly_mul (32-bit p < 2^30, packed rows),
 * through a four-step layout of which only lambda = ceil(lc / n1) rows are
 * transformed: column TFFTs of size lambda, lambda row transforms per
 * operand and for the inverse, and an inverse column TFT (van der Hoeven)
 * that rebuilds each column's lambda coefficients.  For lc just above a
 * power of two this skips about half of the padded transform's row work.
 * Products that fit one pass (lc <= 2^13), and those whose four-step split has
 * columns longer than 2^10 (n = 2^24), go to mm_poly_mul: the same c. */
mm_status mm_poly_mul_tft(uint64_t p, uint64_t g, const uint32_t *a, size_t la, const uint32_t *b, size_t lb,
                          uint32_t *c, size_t batch, void *stream);

/* ------------------------------------------------------------------------
 * Polynomial matrix product: C = A B with A
 * an m x kk and B a kk x n matrix of polynomials over Z/pZ.  A:
 * [m][kk][da] coefficients, B: [kk][n][db], C: [m][n][da + db - 1] (entries
 * row-major, coefficients contiguous, all device memory owned by the
 * caller).  Every entry is transformed once (TFT order, length L =
 * 2^ceil(log2(da + db - 1)), zero padded), the L pointwise m x kk x n
 * matrix products over Z/pZ run on the GPU (exact 64-bit sums, one
 * reduction per entry), and the m n entries of C are transformed back.
 * 32-bit p < 2^30 with 2^log2(L) | p - 1; g generates (Z/pZ)^*.  The
 * library owns an (m kk + kk n + m n) L word workspace per stream;
 * m kk + kk n <= 51200 (MM_E_UNSUPPORTED_SIZE otherwise). */
mm_status mm_poly_matmul(uint64_t p, uint64_t g, const uint32_t *A, const uint32_t *B, uint32_t *C, size_t m,
                         size_t kk, size_t n, size_t da, size_t db, void *stream);

/* ------------------------------------------------------------------------
 * Integer product (P:971-973 Kronecker segmentation, one
 * prime p = 2^64 - 2^32 + 1, R7): a (na limbs) and b (nb limbs)
 * are little-endian 16-bit limbs; c receives exactly na + nb limbs of a b.
 * Exact while min(na, nb) (2^16 - 1)^2 < p (MM_E_SIZE_OVERFLOW otherwise)
 * and na + nb - 1 <= 2^26.  c must not alias a or b. */
mm_status mm_int_mul_u16(const uint16_t *a, size_t na, const uint16_t *b, size_t nb, uint16_t *c,
                         void *stream);

/* ------------------------------------------------------------------------
 * Integer product by the paper's three-prime FFT (SURVEY §8(f)
 * item 1): a (na limbs) and b (nb limbs) are little-endian 32-bit limbs,
 * i.e. Kronecker segmentation with h = 32 (A(2^32) = a).  The three 32-bit
 * NTT products run mod p1 = 998244353, p2 = 985661441, p3 = 943718401
 * (generators 3, 3, 7), the coefficients (< min(na,nb) 2^64 < 2^85 <
 * p1 p2 p3) are rebuilt by Garner's CRT as 96-bit words and carried into c,
 * exactly na + nb limbs.  Transform length <= 2^22 (the 2-adicity of p2, p3),
 * so na + nb - 1 <= 2^22 (MM_E_SIZE_OVERFLOW otherwise).  Device pointers,
 * c must not alias a or b; the library owns its workspace (per stream). */
mm_status mm_int_mul_u32(const uint32_t *a, size_t na, const uint32_t *b, size_t nb, uint32_t *c, void *stream);
/* Integer matrix product (Table 17): C = A B for an m x kk and a
 * kk x n matrix of integers in 32-bit little-endian limbs (A: [m][kk][na],
 * B: [kk][n][nb], C: [m][n][na + nb + 1] -- an entry is a sum of kk
 * products, so it takes one limb more than a product; device memory).  The three-prime
 * method of mm_int_mul_u32 with the pointwise stage a matrix product over
 * each prime (mm_poly_matmul), Garner CRT, carries.  Needs na + nb - 1 <=
 * 2^22 and kk min(na, nb) (2^32 - 1)^2 < p1 p2 p3 (MM_E_SIZE_OVERFLOW). */
mm_status mm_int_matmul_u32(const uint32_t *A, const uint32_t *B, uint32_t *C, size_t m, size_t kk, size_t n,
                            size_t na, size_t nb, void *stream);

/* ------------------------------------------------------------------------
 * Four-step building blocks for the distributed transform (SURVEY a6/a7,
 * Algorithm 1 split across ranks).  The full transform of length n = n2 n1
 * (the plan's n) is viewed as n2 rows x n1 columns, a[j2 n1 + j1].
 * mm_ntt_fwd_cols: Algorithm 1 steps 1-2 on `ncols` consecutive columns
 *   starting at global column col0; `in` holds those columns as an
 *   [n2][ncols] row-major block (natural j2), `out` receives the same shape
 *   with rows in bit-mirrored order i2 (step 1) already multiplied by
 *   w^(j1 [i2]) (step 2).
 * mm_ntt_fwd_rows: Algorithm 1 step 3-4 on `nrows` full rows (length n1)
 *   whose row indices (the bit-mirrored positions i2) start at row0;
 *   in place allowed; output position i2 n1 + i1 = ahat_{[i2 n1 + i1]_k}.
 * mm_ntt_inv_rows / mm_ntt_inv_cols: the inverse steps in reverse order
 *   (inverse row TFFT, multiply by w^(-j1 [i2]); inverse column TFFT and
 *   n^-1), with the same layouts.  Plans must be four-step plans (log2n > 13)
 *   with batch = 1. */
mm_status mm_ntt_fwd_cols(const mm_ntt_plan *plan, const void *in, void *out, size_t col0, size_t ncols,
                          void *stream);
mm_status mm_ntt_fwd_rows(const mm_ntt_plan *plan, const void *in, void *out, size_t row0, size_t nrows,
                          void *stream);
mm_status mm_ntt_inv_rows(const mm_ntt_plan *plan, const void *in, void *out, size_t row0, size_t nrows,
                          void *stream);
mm_status mm_ntt_inv_cols(const mm_ntt_plan *plan, const void *in, void *out, size_t col0, size_t ncols,
                          void *stream);

/* ------------------------------------------------------------------------
 * Many small problems in one launch (BASELINE C1: 16 forward + inverse
 * transforms of 2^10 and one 512 x 512 product).  Each job is one 32-bit
 * problem of length n = 2^k <= 2^12, run by its own CTA of a single kernel
 * launch (the job table is the kernel parameter; nothing is uploaded):
 *   MM_JOB_FORWARD   : out = forward transform of in (P:889 / P:893; `order`
 *                      as mm_ntt_forward), plan = a 32-bit single-pass plan
 *                      (log2n <= 12; its batch is ignored: one row per job).
 *   MM_JOB_INVERSE   : out = inverse of the spectrum in (`order` = order of
 *                      the input, n^-1 included, as mm_ntt_inverse).
 *   MM_JOB_ROUNDTRIP : out = forward(in) in `order` (out may be NULL) and
 *                      out2 = inverse(forward(in)) (BASELINE's
 *                      inverse(forward(x)) = x), the spectrum kept on chip.
 *   MM_JOB_POLY_MUL  : out[0 .. la+lb-2] = in * in2 mod p, in: la
 *                      words, in2: lb words, la + lb - 1 <= 4096; plan NULL,
 *                      (p, g) as mm_poly_mul (p < 2^30, g a generator).
 * Buffers are device memory, residues < p; outputs must not alias another
 * job's buffers (jobs run concurrently).  Asynchronous on `stream`;
 * invalid jobs fail the whole call before anything launches (MM_E_ARG,
 * MM_E_UNSUPPORTED_SIZE).  More than 256 jobs take several launches. */
typedef enum { MM_JOB_FORWARD = 0, MM_JOB_INVERSE = 1, MM_JOB_ROUNDTRIP = 2, MM_JOB_POLY_MUL = 3 } mm_job_kind;
typedef struct {
    int kind;                  /* mm_job_kind */
    int order;                 /* mm_order of the forward output / inverse input */
    const mm_ntt_plan *plan;   /* transform jobs */
    uint64_t p, g;             /* product jobs */
    const void *in, *in2;
    void *out, *out2;
    size_t la, lb;             /* product jobs */
} mm_job;
mm_status mm_run_jobs(const mm_job *jobs, int njobs, void *stream);

/* Sub-batch concurrency of the batched products (default 2): mm_poly_mul /
 * mm_poly_mul_ld with the 2^16-point kernels (C3 shape) split batches of at
 * least 128 n rows into n sub-batches on the library's own streams, forked
 * from and joined back into the caller's stream by events (stream-ordered,
 * no host synchronisation; CUDA-graph capturable), so that one sub-batch's
 * HBM-bound column passes overlap another's ALU-bound product rows.  n = 1
 * runs every kernel on the caller's stream (per-kernel timing).  1 <= n <= 4,
 * else MM_E_ARG.  Process-wide setting. */
mm_status mm_set_product_streams(int n);

/* Free the plans, per-stream workspaces and host-pipeline buffers that
 * mm_poly_mul*, mm_int_mul*, mm_poly_matmul and mm_int_matmul_u32 cache
 * between calls (a cached Goldilocks plan of 2^24 holds 256 MiB of step-2
 * tables, 1 GiB at 2^26) and trim the device's default memory pool.
 * Synchronises the device; no call may be in flight on another host thread.
 * Later calls rebuild what they need. */
mm_status mm_release_cached(void);

/* ------------------------------------------------------------------------
 * Instrumentation (measurement only; not part of the method).
 * mm_launch_count: number of kernels this library has launched in the process.
 * mm_prof_enable(1): clear the profile and bracket every subsequent kernel
 *   launch with CUDA events on its launching stream (0 stops recording).
 * mm_prof_collect: synchronises on the pending events, folds them into the
 *   profile and writes "name launches total_ms\n" lines (aggregated per
 *   kernel family) into buf (truncated to len; buf may be NULL to query the
 *   size); returns the full text length.  Used by bench.py for per-kernel
 *   roofline numbers. */
unsigned long long mm_launch_count(void);
/* Integer-issue probe (ALU roofline of the butterfly): runs the library's own
 * 32-bit (word_bits = 32, radix-16 Shoup/Harvey DIF) or Goldilocks (64,
 * radix-8 FpG::dif; 65: gold.cuh's 8-point split with shift twiddles and
 * delayed reduction) butterfly on register-resident data, `iters` rounds per thread over
 * a full grid, with no memory traffic.  Returns the kernel time (*ms, CUDA
 * events on `stream`, synchronises) and the butterfly count (*bfly). */
mm_status mm_probe_butterfly(int word_bits, int iters, double *ms, double *bfly, void *stream);
/* Instruction-issue probe: 8 independent dependency chains per thread of one
 * SASS class (kind 0 IMAD, 1 IMAD.HI, 2 IADD3, 3 VIADDMNMX, 4 IMAD.HI + 2
 * IADD3 interleaved, 5 DFMA) over a full grid.  Returns the kernel time (*ms) and the
 * warp instructions of that class executed (*ops); ops / (ms x SMs x clock)
 * is the per-SM issue rate that prices each instruction of the butterfly. */
mm_status mm_probe_issue(int kind, int iters, double *ms, double *ops, void *stream);
void mm_prof_enable(int on);
int mm_prof_collect(char *buf, size_t len);

/* Segmented-row variants for the distributed transform (no reshuffle copy):
 * a segmented row block of nrows rows stores element j of row r at
 *   (j / seg_len) * seg_stride + r * seg_len + (j mod seg_len),
 * i.e. n1 / seg_len segments of [nrows][seg_len] each -- exactly the
 * receive buffer of an equal-split all-to-all where segment g came from the
 * rank owning columns [g seg_len, (g+1) seg_len).  seg_len must be a power of
 * two dividing n1 and seg_stride >= nrows * seg_len.
 * mm_ntt_fwd_rows_seg: segmented input -> plain rows output.
 * mm_ntt_inv_rows_seg: plain rows input -> segmented output. */
mm_status mm_ntt_fwd_rows_seg(const mm_ntt_plan *plan, const void *in, void *out, size_t row0, size_t nrows,
                              size_t in_seg_len, size_t in_seg_stride, void *stream);
mm_status mm_ntt_inv_rows_seg(const mm_ntt_plan *plan, const void *in, void *out, size_t row0, size_t nrows,
                              size_t out_seg_len, size_t out_seg_stride, void *stream);

/* Fused column pass + transpose over peer memory (SURVEY §8(e) stretch):
 * Algorithm 1 steps 1-2 on columns [col0, col0 + ncols) of rank `rank` of G,
 * with row t of the block stored straight into peer_recv[t / (n2 / G)] at
 * segment `rank` -- exactly the receive layout of the equal-split
 * all-to-all, so mm_ntt_fwd_rows_seg consumes it unchanged.  peer_recv[h]:
 * G <= 8 device pointers valid in this process (CUDA IPC-opened peer
 * buffers over NVLink, or local buffers), 16-byte aligned.  The caller
 * orders all ranks' writes before the row pass. */
mm_status mm_ntt_fwd_cols_p2p(const mm_ntt_plan *plan, const void *in, void *const *peer_recv, int G, int rank,
                              size_t col0, size_t ncols, void *stream);
/* CUDA IPC plumbing for it: mm_ipc_get_handle writes the 64-byte handle of
 * the cudaMalloc allocation that contains dev_ptr and dev_ptr's byte offset
 * inside it (caching allocators place buffers at offsets); another process
 * of the same node opens the handle (lazy peer access, the allocation base)
 * and adds the offset; mm_ipc_close takes the opened base. */
mm_status mm_ipc_get_handle(const void *dev_ptr, void *handle_out, uint64_t *offset_out);
mm_status mm_ipc_open_handle(const void *handle, void **dev_ptr);
mm_status mm_ipc_close(void *dev_ptr);

/* Sharded integer product blocks (paper_1407_3383_b200/dist.py
 * ShardedIntMul; 64-bit Goldilocks plans):
 *   mm_ntt_fwd_cols_u16 : Algorithm 1 steps 1-2 on columns
 *       [col0, col0 + ncols) of the zero-padded 16-bit limb vector (nlimbs
 *       valid limbs, read in place, widened) viewed as [n2][n1]; out
 *       [n2][ncols] u64.
 *   mm_ntt_pmul_rows_seg : for rows [row0, row0 + nrows) held in segmented
 *       all-to-all buffers (element (r, j) at (j / seg_len) seg_stride +
 *       r seg_len + j mod seg_len) of both operands: steps 3-4, pointwise
 *       product, inverse steps 4-3 and the inverse step-2 twiddle,
 *       into the segmented send buffer c.  No n^-1 (mm_ntt_inv_cols has it).
 * Carries over column blocks (evaluation at 2^16): a rank holds
 * coefficients c_j, j = r n1 + col0 + i for r < nrows, i < c1 (nc product
 * coefficients in all, nout output limbs).  halo[r] = the 4 coefficients
 * before chunk r (from the previous rank; shift = 1 on rank 0, whose row r
 * follows row r - 1 of the last rank).
 *   mm_carry_chunks_halo   : halo_out[r] = last 4 coefficients of chunk r.
 *   mm_carry_chunks_reduce : agg[r] = (generate, propagate) of chunk r.
 *   mm_carry_chunks_scan   : agg_all = all-gathered [G][nrows] aggregates;
 *       replaced in place by the carry into each chunk, chunks taken in
 *       natural order r G + g.
 *   mm_carry_chunks_apply  : out[r][i] = 16-bit limb j of the product. */
mm_status mm_ntt_fwd_cols_u16(const mm_ntt_plan *plan, const uint16_t *limbs, size_t nlimbs, void *out, size_t col0,
                              size_t ncols, void *stream);
mm_status mm_ntt_pmul_rows_seg(const mm_ntt_plan *plan, const void *a, const void *b, void *c, size_t row0,
                               size_t nrows, size_t seg_len, size_t seg_stride, void *stream);
mm_status mm_carry_chunks_halo(const uint64_t *coef, size_t nrows, size_t c1, uint64_t *halo_out, void *stream);
mm_status mm_carry_chunks_reduce(const uint64_t *coef, const uint64_t *halo_in, size_t nrows, size_t c1, size_t n1,
                                 size_t col0, size_t nc, size_t nout, int shift, uint32_t *agg, void *stream);
mm_status mm_carry_chunks_scan(uint32_t *agg_all, size_t G, size_t nrows, void *stream);
mm_status mm_carry_chunks_apply(const uint64_t *coef, const uint64_t *halo_in, size_t nrows, size_t c1, size_t n1,
                                size_t col0, size_t nc, size_t nout, int shift, const uint32_t *cin, uint16_t *out,
                                void *stream);


/* ------------------------------------------------------------------------
 * Distributed transform and integer product (Algorithm 1
 * split across the GPUs of one node: "a critical point in large
 * sizes becomes the matrix transposition", P:925 -- here an all-to-all).
 * One process per GPU.  NCCL is not linked: libnccl.so.2 is dlopen'ed (the
 * copy torch already loaded), MM_E_NCCL if it cannot be.
 *   mm_dist_unique_id : 128-byte NCCL unique id (rank 0; the caller
 *       broadcasts it, e.g. over torch.distributed).
 *   mm_dist_create    : communicator of `world` <= 8 ranks on the current
 *       device; *d owned by the library (mm_dist_destroy).  Collective.
 *   mm_dist_info      : out = {rank, world, p2p receive-buffer bytes (0 = NCCL
 *       transport), NCCL version code}.
 *   mm_dist_p2p_enable: setup (collective, synchronises): two receive buffers
 *       of `bytes` and a flag page in one cudaMalloc, IPC handles all-gathered,
 *       peers opened.  Afterwards mm_ntt_forward_dist uses the fused transpose
 *       (mm_ntt_fwd_cols_p2p stores rows into the peers' receive buffers over
 *       NVLink) ordered by device-side flags (release / acquire at system
 *       scope), no all-to-all and no host barrier, whenever a column block
 *       fits `bytes`.
 *   mm_dist_p2p_status: 0, or 1 + the flag slot of a device-side wait that
 *       timed out (~20 s: a peer stopped); synchronises the device.
 * Plans: four-step (log2n > 13), batch 1, with n1 and
 * n2 divisible by world.  Rank g of G, c1 = n1 / G, r2 = n2 / G:
 *   mm_ntt_forward_dist : local_in = [n2][c1] column block (natural input
 *       element j2 n1 + j1, j1 in [g c1, (g+1) c1)); local_out = [r2][n1] row
 *       block = positions [g r2 n1, (g+1) r2 n1) of the TFT-order output
 *       (position i holds ahat_{[i]_k}).
 *   mm_ntt_inverse_dist : the reverse (row block in, column block out, n^-1).
 *   mm_int_mul_u16_dist : a (na limbs), b (nb limbs) whole on every rank (2 B
 *       per limb); the product of mm_int_mul_u16 with one all-to-all per
 *       operand and one back, carries by a ring halo exchange and an
 *       all-gather of per-chunk (generate, propagate) pairs; local_c =
 *       [n2][c1] limbs, element (r, i) = limb r n1 + g c1 + i of a b (0 beyond
 *       na + nb).  mm_int_mul_u16_dist_layout gives {n1, n2, c1, log2 n}.
 * Workspaces are stream-ordered allocations; all calls are asynchronous on
 * `stream` and collective (every rank calls them in the same order). */
typedef struct mm_dist mm_dist;
mm_status mm_dist_unique_id(void *id_out);
mm_status mm_dist_create(const void *nccl_unique_id, int rank, int world, mm_dist **d);
void mm_dist_destroy(mm_dist *d);
mm_status mm_dist_info(const mm_dist *d, int64_t out[4]);
mm_status mm_dist_p2p_enable(mm_dist *d, size_t bytes);
mm_status mm_dist_p2p_status(mm_dist *d, uint64_t *slot);
mm_status mm_ntt_forward_dist(mm_dist *d, const mm_ntt_plan *plan, const void *local_in, void *local_out,
                              void *stream);
mm_status mm_ntt_inverse_dist(mm_dist *d, const mm_ntt_plan *plan, const void *local_in, void *local_out,
                              void *stream);
mm_status mm_int_mul_u16_dist(mm_dist *d, const uint16_t *a, size_t na, const uint16_t *b, size_t nb,
                              uint16_t *local_c, void *stream);
mm_status mm_int_mul_u16_dist_layout(mm_dist *d, size_t na, size_t nb, uint64_t out[4]);

#ifdef __cplusplus
}
#endif
#endif /* MMNTT_H */
