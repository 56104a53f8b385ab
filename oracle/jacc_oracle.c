/*
 * jacc_oracle.c -- the CPU ORACLE for the Jacc hot path.  TEST INFRASTRUCTURE.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product path
 * (paper_1508_06791_b200/, libjacc.so) never links, imports or calls it, and
 * the two share no code: no headers, no helpers, no constants tables.
 *
 * Plain, slow, obviously correct loops, in the order the definitions are
 * written.  Floating point is accumulated in fp64 (the north_star's
 * "fp64-accumulated oracle"), except vector add, whose definition IS one
 * IEEE fp32 add.  Built with `gcc -O2 -fno-fast-math -ffp-contract=off`
 * (no FMA contraction, no reassociation); OpenMP only over independent
 * outer indices, so results do not depend on the thread count.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; SURVEY §8(c) holds the
 * readings (ambiguities) each function follows, listed again in DESIGN.md.
 *
 * Pins: every function here is pinned by tests/test_oracle_pins.py against
 * something other than itself (closed forms, brute force, invariants,
 * library routines).  None is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* Thread count of the OpenMP loops below (bench.py's single-thread vs
 * all-core CPU baseline); results never depend on it. */
void oracle_set_num_threads(int n) {
#ifdef _OPENMP
    omp_set_num_threads(n > 0 ? n : 1);
#else
    (void)n;
#endif
}

/* ---------------------------------------------------------------------
 * Vector addition ("performs the addition of two ... vectors").
 * c[i] = fl32(a[i] + b[i]): one IEEE-754 binary32 round-to-nearest add.
 * ------------------------------------------------------------------- */
void oracle_vadd_f32(const float *a, const float *b, float *c, int64_t n) {
    for (int64_t i = 0; i < n; ++i) {
        float s = a[i] + b[i]; /* SSE scalar add, FLT_EVAL_METHOD == 0 */
        c[i] = s;
    }
}

/* ---------------------------------------------------------------------
 * Reduction: "performs a summation across an array";
 * the @Atomic(op=ADD) field turns the assignment into `result += sum`
 * (P:140), and is auto-initialised to zero.
 * s = init + sum_i x[i], accumulated sequentially in fp64.  Also returns
 * sum_i |x[i]| (the scale the tolerance gate is expressed in, DESIGN R14).
 * ------------------------------------------------------------------- */
double oracle_reduce_sum_f32(const float *x, int64_t n, double init, double *abs_sum) {
    double s = init;
    double a = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        s += (double)x[i];
        a += fabs((double)x[i]);
    }
    if (abs_sum) *abs_sum = a;
    return s;
}

/* ---------------------------------------------------------------------
 * Histogram: "produces frequency counts for ... values,
 * placing the results into 256 distinct bins"; bins are an @Atomic ADD
 * output (Table 1).  bins[k] (+)= #{i : keys[i] == k}, 0 <= k < nbins.
 * Reading R11: keys outside [0, nbins) are ignored.  accumulate == 0 is
 * the WRITE mode (auto-zero first); accumulate != 0 is READWRITE.
 * ------------------------------------------------------------------- */
void oracle_histogram_i32(const int32_t *keys, int64_t n, int32_t nbins,
                          int32_t *bins, int accumulate) {
    if (!accumulate)
        for (int32_t k = 0; k < nbins; ++k) bins[k] = 0;
    for (int64_t i = 0; i < n; ++i) {
        int32_t k = keys[i];
        if (k >= 0 && k < nbins) bins[k] += 1;
    }
}

/* ---------------------------------------------------------------------
 * Black-Scholes ("an implementation of the Black Scholes option
 * pricing model ... supplied as an example in the APARAPI source code").
 * Reading R12: the APARAPI sample's formula:
 *   phi(x) = y if x >= 0 else 1 - y,
 *   t = 1/(1 + 0.2316419|x|),
 *   y = 1 - 0.398942280 exp(-x^2/2) t (c1 + t(c2 + t(c3 + t(c4 + t c5))))
 *   d1 = (ln(S/K) + (R + sigma^2/2) T) / (sigma sqrt T),  d2 = d1 - sigma sqrt T
 *   call = S phi(d1) - K e^{-RT} phi(d2);  put = K e^{-RT} phi(-d2) - S phi(-d1)
 * computed in fp64 from the fp32 inputs (exactly widened).
 * ------------------------------------------------------------------- */
double oracle_bs_phi(double x) {
    const double c1 = 0.319381530, c2 = -0.356563782, c3 = 1.781477937,
                 c4 = -1.821255978, c5 = 1.330274429;
    double ax = fabs(x);
    double t = 1.0 / (1.0 + 0.2316419 * ax);
    double poly = c1 + t * (c2 + t * (c3 + t * (c4 + t * c5)));
    double y = 1.0 - 0.398942280 * exp(-x * x / 2.0) * t * poly;
    return (x < 0.0) ? (1.0 - y) : y;
}

void oracle_bs_price(double S, double K, double T, double R, double sigma,
                     double *call, double *put) {
    double sigma_sqrt_t = sigma * sqrt(T);
    double d1 = (log(S / K) + (R + sigma * sigma / 2.0) * T) / sigma_sqrt_t;
    double d2 = d1 - sigma_sqrt_t;
    double k_exp_mrt = K * exp(-R * T);
    *call = S * oracle_bs_phi(d1) - k_exp_mrt * oracle_bs_phi(d2);
    *put = k_exp_mrt * oracle_bs_phi(-d2) - S * oracle_bs_phi(-d1);
}

/* APARAPI mapping of one uniform draw u in [0,1) to the option parameters:
 * X = X_lo * u + X_hi * (1 - u), with S, K in [10, 100], T in [1, 10],
 * R in [0.01, 0.05], sigma in [0.01, 0.10]. */
void oracle_bs_params(double u, double *S, double *K, double *T, double *R, double *sigma) {
    *S = 10.0 * u + 100.0 * (1.0 - u);
    *K = 10.0 * u + 100.0 * (1.0 - u);
    *T = 1.0 * u + 10.0 * (1.0 - u);
    *R = 0.01 * u + 0.05 * (1.0 - u);
    *sigma = 0.01 * u + 0.10 * (1.0 - u);
}

void oracle_blackscholes_f32(const float *rnd, int64_t n, double *call, double *put) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double S, K, T, R, sigma;
        oracle_bs_params((double)rnd[i], &S, &K, &T, &R, &sigma);
        oracle_bs_price(S, K, T, R, sigma, &call[i], &put[i]);
    }
}

void oracle_blackscholes_soa_f32(const float *S, const float *K, const float *T,
                                 const float *R, const float *sigma, int64_t n,
                                 double *call, double *put) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        oracle_bs_price((double)S[i], (double)K[i], (double)T[i], (double)R[i],
                        (double)sigma[i], &call[i], &put[i]);
}

/* ---------------------------------------------------------------------
 * Dense matrix multiply (SGEMM).  Reading R13: row-major,
 * C = A.B (beta = 0).  C[r][j] = sum_{k=0}^{K-1} A[r][k] B[k][j], each
 * product and the running sum in fp64 (products of two fp32 are exact in
 * fp64).  Computed for the requested rows only (rows == NULL: all M rows).
 * ------------------------------------------------------------------- */
void oracle_sgemm_rows_f32(const float *A, const float *B, double *C,
                           int64_t M, int64_t N, int64_t K,
                           int64_t lda, int64_t ldb, int64_t ldc,
                           const int64_t *rows, int64_t nrows) {
    int64_t cnt = rows ? nrows : M;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t ri = 0; ri < cnt; ++ri) {
        int64_t r = rows ? rows[ri] : ri;
        double *c = C + ri * ldc;
        for (int64_t j = 0; j < N; ++j) c[j] = 0.0;
        /* k outer, j inner: every c[j] still accumulates k = 0, 1, ..., K-1
         * in order -- the definition's order -- with a streaming inner loop. */
        for (int64_t k = 0; k < K; ++k) {
            double a = (double)A[r * lda + k];
            const float *b = B + k * ldb;
            for (int64_t j = 0; j < N; ++j) c[j] += a * (double)b[j];
        }
    }
}

/* ---------------------------------------------------------------------
 * N-body (north_star only; not in the paper -- SURVEY D1, reading R16).
 * Direct-sum softened gravity:
 *   a_i = G sum_j m_j (x_j - x_i) / (|x_j - x_i|^2 + eps2)^{3/2}
 * (the self term j == i contributes exactly 0 because eps2 > 0).
 * pos: n_src x 4 doubles (x, y, z, m).  Accelerations of the targets tgt[]
 * are written to acc (n_tgt x 3).
 * ------------------------------------------------------------------- */
void oracle_nbody_accel(const double *pos, int64_t n_src, const int64_t *tgt,
                        int64_t n_tgt, double eps2, double G, double *acc) {
#pragma omp parallel for schedule(static)
    for (int64_t t = 0; t < n_tgt; ++t) {
        int64_t i = tgt[t];
        double xi = pos[4 * i + 0], yi = pos[4 * i + 1], zi = pos[4 * i + 2];
        double ax = 0.0, ay = 0.0, az = 0.0;
        for (int64_t j = 0; j < n_src; ++j) {
            double dx = pos[4 * j + 0] - xi;
            double dy = pos[4 * j + 1] - yi;
            double dz = pos[4 * j + 2] - zi;
            double r2 = dx * dx + dy * dy + dz * dz + eps2;
            double inv_r3 = 1.0 / (r2 * sqrt(r2));
            double s = pos[4 * j + 3] * inv_r3;
            ax += dx * s;
            ay += dy * s;
            az += dz * s;
        }
        acc[3 * t + 0] = G * ax;
        acc[3 * t + 1] = G * ay;
        acc[3 * t + 2] = G * az;
    }
}

/* Symplectic (semi-implicit) Euler, `steps` times, on the whole system:
 *   a = accel(x);  v <- v + a dt;  x <- x + v dt.
 * pos (n x 4: x, y, z, m) and vel (n x 4: vx, vy, vz, 0) are updated in
 * place in fp64.  scratch: n x 3 doubles, tgt: 0..n-1. */
void oracle_nbody_steps(double *pos, double *vel, int64_t n, int steps,
                        double dt, double eps2, double G,
                        double *scratch, const int64_t *tgt) {
    for (int s = 0; s < steps; ++s) {
        oracle_nbody_accel(pos, n, tgt, n, eps2, G, scratch);
        for (int64_t i = 0; i < n; ++i) {
            vel[4 * i + 0] += scratch[3 * i + 0] * dt;
            vel[4 * i + 1] += scratch[3 * i + 1] * dt;
            vel[4 * i + 2] += scratch[3 * i + 2] * dt;
            pos[4 * i + 0] += vel[4 * i + 0] * dt;
            pos[4 * i + 1] += vel[4 * i + 1] * dt;
            pos[4 * i + 2] += vel[4 * i + 2] * dt;
        }
    }
}

/* ---------------------------------------------------------------------
 * 2D convolution ("convolves a 2048 x 2048
 * image with a 5 x 5 filter").  Reading R20: true convolution (the filter
 * is flipped), zero padding outside the image, output the size of the image:
 *   out[y][x] = sum_{i=0}^{2r} sum_{j=0}^{2r} f[i][j] img[y + r - i][x + r - j]
 * accumulated in fp64 over i then j.  Also returns, per output, the scale
 * sum |f[i][j]| |img[...]| the tolerance is expressed in (abs_out may be NULL).
 * ------------------------------------------------------------------- */
void oracle_conv2d_f32(const float *img, int64_t H, int64_t W, const float *f, int r,
                       double *out, double *abs_out) {
    const int k = 2 * r + 1;
#pragma omp parallel for schedule(static)
    for (int64_t y = 0; y < H; ++y) {
        for (int64_t x = 0; x < W; ++x) {
            double s = 0.0, a = 0.0;
            for (int i = 0; i < k; ++i) {
                const int64_t yy = y + r - i;
                if (yy < 0 || yy >= H) continue;
                for (int j = 0; j < k; ++j) {
                    const int64_t xx = x + r - j;
                    if (xx < 0 || xx >= W) continue;
                    const double p = (double)f[i * k + j] * (double)img[yy * W + xx];
                    s += p;
                    a += fabs(p);
                }
            }
            out[y * W + x] = s;
            if (abs_out) abs_out[y * W + x] = a;
        }
    }
}

/* ---------------------------------------------------------------------
 * Correlation matrix ("the Lucene OpenBitSet
 * 'intersection count' ... 1024 Terms and 16384 Documents"; "popc").
 * Reading R21: term t is a bitset over the documents, stored as `words`
 * 32-bit words (bit d%32 of word d/32 = document d);
 *   C[i][j] = #{documents in both A_i and B_j} = sum_w popcount(A_i[w] & B_j[w]).
 * Bits are counted one by one (no builtin), the literal definition.
 * ------------------------------------------------------------------- */
void oracle_corr_popc(const uint32_t *A, int64_t ta, const uint32_t *B, int64_t tb,
                      int64_t words, int32_t *C) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < ta; ++i)
        for (int64_t j = 0; j < tb; ++j) {
            int64_t c = 0;
            for (int64_t w = 0; w < words; ++w) {
                uint32_t v = A[i * words + w] & B[j * words + w];
                for (int b = 0; b < 32; ++b) c += (v >> b) & 1u;
            }
            C[i * tb + j] = (int32_t)c;
        }
}

/* ---------------------------------------------------------------------
 * Sparse matrix-vector multiply, CSR ("a 44609 x
 * 44609 matrix with 1029655 non-zeros (The bcsstk32 matrix from Matrix
 * Market)").  Reading R22: y = A x, A in CSR (row_ptr[n+1], col[nnz],
 * val[nnz]); y[i] = sum_{k=row_ptr[i]}^{row_ptr[i+1]-1} val[k] x[col[k]] in
 * fp64 in k order; abs_out[i] = sum |val[k] x[col[k]]| (tolerance scale).
 * ------------------------------------------------------------------- */
void oracle_spmv_csr_f32(const int32_t *row_ptr, const int32_t *col, const float *val,
                         const float *x, int64_t n, double *y, double *abs_out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0, a = 0.0;
        for (int64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
            double p = (double)val[k] * (double)x[col[k]];
            s += p;
            a += fabs(p);
        }
        y[i] = s;
        if (abs_out) abs_out[i] = a;
    }
}
