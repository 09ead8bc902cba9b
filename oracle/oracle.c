/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY.  The plain, slow, obviously-correct CPU
 * oracle for C += A.B with F16 inputs (arXiv 2108.13191).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
 * leg may load this library.  The product path (paper_2108_13191_b200/) never
 * does, and shares no code, header, table or constant with this file.
 *
 * What it computes (PAPER.md, cited as P:<line>):
 *   - Problem statement, Sec. 4: "a matmul of the form C = AB + C
 *     (all three matrices are stored in a row-major layout)".
 *   - Starting point, Sec. 3.1 P:412-418 / Listing lst:naive-affine P:420-438:
 *     the three-loop nest C[i][j] += A[i][k] * B[k][j].
 *   - Algorithm 1: the same sum, tiled; tiling does not change the
 *     definition, so the oracle is the untiled loop nest.
 *   - Precisions, Sec. 4.1 P:926-930 (F16 inputs, F32 accumulate and output)
 *     and Sec. 4.2 P:976-980 (F16 inputs, F16 accumulate and output).
 *
 * Arithmetic: every element is evaluated as
 *     x_ij = C_in[i][j] + sum_{k=0}^{K-1} A[i][k] * B[k][j]
 * in IEEE double with k ascending (loop order i-k-j with one double accumulator
 * per element of the current row, so each element still sums k ascending).
 * Products of two binary16 values are exact in double (11+11 significant bits);
 * only the additions round, which bounds |x_ij - exact| by
 * gamma_K * sum_k |a_ik b_kj| + ..., gamma_K = K u/(1-K u), u = 2^-53.
 * Rounding to the output type is done once, RNE (readings R3, R5):
 *   F32 output: (float)x  -- C's double->float conversion, round-to-nearest-even.
 *   F16 output: oracle_f64_to_f16_rne() below (own encoder, RNE, overflow -> Inf).
 *
 * Parallelism: OpenMP over rows i only, so results are bitwise independent of
 * the thread count.  Build with -ffp-contract=off so no FMA contraction changes
 * the rounding of the accumulation.
 *
 * Pins (tests/test_oracle_pins.py): exact rationals on tiny shapes, numpy
 * float64 on 256^3, closed forms (identity, permutation, zero, all-ones = K,
 * rank-1 powers of two, small integers), all 65536 binary16 patterns for the
 * decoder, numpy's binary16 rounding for the encoder.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* IEEE 754 binary16 -> double, exact.  1 sign bit, 5 exponent bits (bias 15),
 * 10 fraction bits.  e == 0: subnormal f * 2^-24; e == 31: Inf / NaN. */
double oracle_f16_to_f64(uint16_t h)
{
    int sign = (h >> 15) & 1;
    int e = (h >> 10) & 0x1f;
    int f = h & 0x3ff;
    double v;
    if (e == 0) {
        v = ldexp((double)f, -24);
    } else if (e == 31) {
        v = (f == 0) ? INFINITY : NAN;
    } else {
        v = ldexp((double)(f | 0x400), e - 25);
    }
    return sign ? -v : v;
}

/* double -> binary16, round to nearest, ties to even.  Overflow -> +-Inf (no
 * saturation, R5), NaN -> quiet NaN 0x7e00 with the sign kept. */
uint16_t oracle_f64_to_f16_rne(double x)
{
    uint16_t sign = signbit(x) ? 0x8000 : 0;
    if (isnan(x)) return (uint16_t)(sign | 0x7e00);
    double a = fabs(x);
    if (isinf(a)) return (uint16_t)(sign | 0x7c00);
    if (a == 0.0) return sign;
    /* Quantum of the binary16 grid around a: normal numbers with exponent E
     * (2^E <= a < 2^(E+1), E >= -14) have spacing 2^(E-10); subnormals and the
     * smallest binade share spacing 2^-24. */
    int E;
    frexp(a, &E);          /* a = m * 2^E, 0.5 <= m < 1, so 2^(E-1) <= a < 2^E */
    E -= 1;                /* now 2^E <= a < 2^(E+1) */
    if (E < -14) E = -14;
    double q = ldexp(1.0, E - 10);
    double n = a / q;      /* exact: q is a power of two and n < 2^11 fits */
    double fl = floor(n);
    double r = n - fl;
    double m;
    if (r > 0.5) m = fl + 1.0;
    else if (r < 0.5) m = fl;
    else m = (fmod(fl, 2.0) == 0.0) ? fl : fl + 1.0;
    double v = m * q;      /* rounded magnitude, exact in double */
    if (v > 65504.0) return (uint16_t)(sign | 0x7c00);
    /* encode v exactly */
    if (v < ldexp(1.0, -14)) {                       /* subnormal (or 2^-14 boundary) */
        uint16_t f = (uint16_t)(v / ldexp(1.0, -24));
        return (uint16_t)(sign | f);                  /* f == 1024 encodes 2^-14 */
    }
    int Ev;
    double mv = frexp(v, &Ev);                        /* v = mv * 2^Ev */
    int e = Ev - 1 + 15;                              /* biased exponent */
    uint16_t f = (uint16_t)((mv * 2.0 - 1.0) * 1024.0);
    return (uint16_t)(sign | (e << 10) | f);
}

/* bfloat16 -> double, exact: bfloat16 is the top half of an IEEE binary32
 * (1 sign bit, 8 exponent bits with bias 127, 7 fraction bits).  Decoded from
 * the fields, not by reinterpreting memory.  PAPER.md Sec. 2.3 P:272-275 lists
 * BF16 among the tensor-core input formats. */
double oracle_bf16_to_f64(uint16_t h)
{
    int sign = (h >> 15) & 1;
    int e = (h >> 7) & 0xff;
    int f = h & 0x7f;
    double v;
    if (e == 0) {
        v = ldexp((double)f, -133);                 /* subnormal: f * 2^(1-127-7) */
    } else if (e == 255) {
        v = (f == 0) ? INFINITY : NAN;
    } else {
        v = ldexp((double)(f | 0x80), e - 134);     /* (1.f) * 2^(e-127), f has 7 bits */
    }
    return sign ? -v : v;
}

/* acc_type: 0 = F32 (C is float), 1 = F16 (C is binary16 bits). */
static double load_c(const void* C, int64_t idx, int acc_type)
{
    if (acc_type == 0) return (double)((const float*)C)[idx];
    return oracle_f16_to_f64(((const uint16_t*)C)[idx]);
}

/*
 * oracle_gemm_f16: the definition, row by row.
 *   M, N, K        problem extents (>= 0)
 *   A, lda         binary16 bits, row-major M x K, element (i,k) at A[i*lda + k]
 *   B, ldb         binary16 bits, row-major K x N, element (k,j) at B[k*ldb + j]
 *   C_in, ldc      acc_type elements, row-major M x N (the "+ C" of P:908)
 *   acc_type       0 = F32 accumulate/output, 1 = F16 accumulate/output
 *   rows, nrows    rows of the result to compute (NULL: all M rows, nrows = M)
 *   C_exact        out, double, nrows x N, row r at C_exact[r*N]   (may be NULL)
 *   C_round        out, acc_type, nrows x N, row r at r*N           (may be NULL)
 * Returns 0, or -1 on an invalid argument (negative extent, short ld,
 * out-of-range row index).
 */
/*
 * oracle_gemm_ex: the fused-epilogue generalisation (the
 * paper's motivation for fusion):
 *     x_ij = beta * C_in[i][j] + sum_k A[i][k] * B[k][j] + bias[j]
 *     out_ij = relu ? (x_ij > 0 ? x_ij : (x_ij is NaN ? x_ij : 0)) : x_ij
 * evaluated in IEEE double (C_in first, then k ascending, then the bias), then
 * rounded once to the output type.  in_type: 0 = binary16 A/B, 1 = bfloat16.
 * beta: 0 or 1 (beta = 0 ignores C_in, which is then not read).  bias: NULL or
 * N floats.  With in_type 0, beta 1, no bias, no relu this is oracle_gemm_f16.
 */
int oracle_gemm_ex(int64_t M, int64_t N, int64_t K,
                   const uint16_t* A, int64_t lda,
                   const uint16_t* B, int64_t ldb,
                   const void* C_in, int64_t ldc,
                   int acc_type, int in_type, int beta, const float* bias, int relu,
                   const int64_t* rows, int64_t nrows,
                   double* C_exact, void* C_round);

int oracle_gemm_f16(int64_t M, int64_t N, int64_t K,
                    const uint16_t* A, int64_t lda,
                    const uint16_t* B, int64_t ldb,
                    const void* C_in, int64_t ldc,
                    int acc_type,
                    const int64_t* rows, int64_t nrows,
                    double* C_exact, void* C_round)
{
    return oracle_gemm_ex(M, N, K, A, lda, B, ldb, C_in, ldc, acc_type, 0, 1, NULL, 0, rows, nrows,
                          C_exact, C_round);
}

int oracle_gemm_ex(int64_t M, int64_t N, int64_t K,
                   const uint16_t* A, int64_t lda,
                   const uint16_t* B, int64_t ldb,
                   const void* C_in, int64_t ldc,
                   int acc_type, int in_type, int beta, const float* bias, int relu,
                   const int64_t* rows, int64_t nrows,
                   double* C_exact, void* C_round)
{
    if (in_type != 0 && in_type != 1) return -1;
    if (beta != 0 && beta != 1) return -1;
    double (*decode)(uint16_t) = in_type == 0 ? oracle_f16_to_f64 : oracle_bf16_to_f64;
    if (M < 0 || N < 0 || K < 0) return -1;
    if (acc_type != 0 && acc_type != 1) return -1;
    if (K > 0 && lda < K) return -1;
    if (N > 0 && (ldb < N || ldc < N)) return -1;
    if (rows == NULL) nrows = M;
    for (int64_t r = 0; rows != NULL && r < nrows; ++r)
        if (rows[r] < 0 || rows[r] >= M) return -1;
    if (N == 0 || nrows == 0) return 0;

    /* Decode B once (exact: binary16 values are exactly representable in double). */
    double* Bd = (double*)malloc((size_t)(K > 0 ? K : 1) * (size_t)N * sizeof(double));
    if (!Bd) return -2;
    for (int64_t k = 0; k < K; ++k)
        for (int64_t j = 0; j < N; ++j)
            Bd[k * N + j] = decode(B[k * ldb + j]);

    int status = 0;
#pragma omp parallel
    {
        double* acc = (double*)malloc((size_t)N * sizeof(double));
        if (!acc) {
#pragma omp atomic write
            status = -2;
        }
#pragma omp for schedule(dynamic, 1)
        for (int64_t r = 0; r < nrows; ++r) {
            if (!acc) continue;
            int64_t i = rows ? rows[r] : r;
            /* x_ij starts at C_in[i][j] (C = AB + C), or at 0 when beta = 0 */
            for (int64_t j = 0; j < N; ++j) acc[j] = beta ? load_c(C_in, i * ldc + j, acc_type) : 0.0;
            /* k ascending: x_ij += A[i][k] * B[k][j]  (lst:naive-affine) */
            for (int64_t k = 0; k < K; ++k) {
                double a = decode(A[i * lda + k]);
                const double* brow = Bd + k * N;
                for (int64_t j = 0; j < N; ++j) acc[j] += a * brow[j];
            }
            if (bias)   /* + bias[j], broadcast over rows */
                for (int64_t j = 0; j < N; ++j) acc[j] += (double)bias[j];
            if (relu)   /* max(x, 0), NaN propagates */
                for (int64_t j = 0; j < N; ++j)
                    if (!(acc[j] > 0.0) && !isnan(acc[j])) acc[j] = 0.0;
            if (C_exact) memcpy(C_exact + r * N, acc, (size_t)N * sizeof(double));
            if (C_round) {
                if (acc_type == 0) {
                    float* out = (float*)C_round + r * N;
                    for (int64_t j = 0; j < N; ++j) out[j] = (float)acc[j];
                } else {
                    uint16_t* out = (uint16_t*)C_round + r * N;
                    for (int64_t j = 0; j < N; ++j) out[j] = oracle_f64_to_f16_rne(acc[j]);
                }
            }
        }
        free(acc);
    }
    free(Bd);
    return status;
}

/* Threads the OpenMP runtime will use (reported beside the oracle's timing). */
int oracle_num_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
