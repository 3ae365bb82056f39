/*
 * TEST INFRASTRUCTURE ONLY -- CPU oracle, "fast" GEMM family.
 *
 * Restates the reference's fast kernel (rnnblock kernels.py:98-178): output
 * rows in chunks of 128 (_ROW_CHUNK, kernels.py:112) split over worker
 * threads (numba prange -> OpenMP here), columns in register panels of
 * 8/4/2/1 (kernels.py:136-178) reading B transposed so every inner loop is
 * unit stride, reassociation allowed (numba fastmath -> -ffast-math here).
 * Each output element is produced by exactly one thread, so results do not
 * depend on the thread count (kernels.py:101-110).
 *
 * This is the CPU baseline bench.py times ("cpu_baseline", kind "port") and
 * the fast leg of the oracle.  Never part of the product path.
 */
#include <math.h>
#include <stdint.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ROW_CHUNK 128

void orc_set_threads(int n)
{
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_get_threads(void)
{
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ISA: the Makefile builds an AVX-512 (x86-64-v4) and an AVX2 (x86-64-v3)
   library; oracle.py loads the one the host supports (numba's LLVM likewise
   targets the host ISA). */
#define ORC_CLONES

#define FAST_DEFINE(T, SFX)                                                               \
    ORC_CLONES void orc_gemm_fast_##SFX(const T *A, const T *Bt, T *C, int64_t m, int64_t k,        \
                             int64_t n)                                                   \
    {                                                                                     \
        int64_t nchunks = (m + ROW_CHUNK - 1) / ROW_CHUNK;                                \
        int64_t n8 = (n / 8) * 8;                                                         \
        _Pragma("omp parallel for schedule(static) if(nchunks > 1)")                      \
        for (int64_t ci = 0; ci < nchunks; ++ci) {                                        \
            int64_t i0 = ci * ROW_CHUNK, i1 = i0 + ROW_CHUNK < m ? i0 + ROW_CHUNK : m;     \
            for (int64_t j0 = 0; j0 < n8; j0 += 8)                                        \
                for (int64_t i = i0; i < i1; ++i) {                                       \
                    const T *a = A + i * k;                                               \
                    const T *b0 = Bt + j0 * k;                                            \
                    T s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0, s6 = 0, s7 = 0;     \
                    for (int64_t p = 0; p < k; ++p) {                                     \
                        T av = a[p];                                                      \
                        s0 += av * b0[p];                                                 \
                        s1 += av * b0[k + p];                                             \
                        s2 += av * b0[2 * k + p];                                         \
                        s3 += av * b0[3 * k + p];                                         \
                        s4 += av * b0[4 * k + p];                                         \
                        s5 += av * b0[5 * k + p];                                         \
                        s6 += av * b0[6 * k + p];                                         \
                        s7 += av * b0[7 * k + p];                                         \
                    }                                                                     \
                    T *c = C + i * n + j0;                                                \
                    c[0] = s0; c[1] = s1; c[2] = s2; c[3] = s3;                           \
                    c[4] = s4; c[5] = s5; c[6] = s6; c[7] = s7;                           \
                }                                                                         \
            int64_t j0 = n8;                                                              \
            if (j0 + 4 <= n) {                                                            \
                for (int64_t i = i0; i < i1; ++i) {                                       \
                    const T *a = A + i * k, *b0 = Bt + j0 * k;                            \
                    T s0 = 0, s1 = 0, s2 = 0, s3 = 0;                                     \
                    for (int64_t p = 0; p < k; ++p) {                                     \
                        T av = a[p];                                                      \
                        s0 += av * b0[p];                                                 \
                        s1 += av * b0[k + p];                                             \
                        s2 += av * b0[2 * k + p];                                         \
                        s3 += av * b0[3 * k + p];                                         \
                    }                                                                     \
                    T *c = C + i * n + j0;                                                \
                    c[0] = s0; c[1] = s1; c[2] = s2; c[3] = s3;                           \
                }                                                                         \
                j0 += 4;                                                                  \
            }                                                                             \
            if (j0 + 2 <= n) {                                                            \
                for (int64_t i = i0; i < i1; ++i) {                                       \
                    const T *a = A + i * k, *b0 = Bt + j0 * k;                            \
                    T s0 = 0, s1 = 0;                                                     \
                    for (int64_t p = 0; p < k; ++p) {                                     \
                        s0 += a[p] * b0[p];                                               \
                        s1 += a[p] * b0[k + p];                                           \
                    }                                                                     \
                    C[i * n + j0] = s0; C[i * n + j0 + 1] = s1;                           \
                }                                                                         \
                j0 += 2;                                                                  \
            }                                                                             \
            if (j0 < n) {                                                                 \
                for (int64_t i = i0; i < i1; ++i) {                                       \
                    const T *a = A + i * k, *b0 = Bt + j0 * k;                            \
                    T s0 = 0;                                                             \
                    for (int64_t p = 0; p < k; ++p) s0 += a[p] * b0[p];                   \
                    C[i * n + j0] = s0;                                                   \
                }                                                                         \
            }                                                                             \
        }                                                                                 \
    }

FAST_DEFINE(float, f32)
FAST_DEFINE(double, f64)

/* Elementwise phases of the fast path, parallel + SIMD like the reference's
 * numpy ufuncs (kernels.py:236-241, blocked.py:129-130,144-149) and its
 * prange sweep (blocked.py:153-162).  glibc's libmvec supplies vector tanh. */
#define FAST_ELEM(T, SFX, TANH)                                                            \
    ORC_CLONES void orc_sig_bias_fast_##SFX(T *g, const T *b, int64_t dh, int64_t l)       \
    {                                                                                      \
        _Pragma("omp parallel for schedule(static) if(dh * l > 2048)")                    \
        for (int64_t i = 0; i < dh; ++i) {                                                 \
            T bi = b[i];                                                                   \
            _Pragma("omp simd")                                                            \
            for (int64_t t = 0; t < l; ++t)                                                \
                g[i * l + t] = (T)0.5 * ((T)1 + TANH((T)0.5 * (g[i * l + t] + bi)));       \
        }                                                                                  \
    }                                                                                      \
    /* row-parallel so the SIMD/remainder split of every row is independent of   */ \
    /* the thread count (results must not depend on it, kernels.py:101-110)       */ \
    ORC_CLONES void orc_tap_act_fast_##SFX(T *g, const T *tmp, int64_t dh, int64_t l,      \
                                           int is_tanh)                                    \
    {                                                                                      \
        _Pragma("omp parallel for schedule(static) if(dh * l > 2048)")                    \
        for (int64_t i = 0; i < dh; ++i) {                                                 \
            _Pragma("omp simd")                                                            \
            for (int64_t t = 0; t < l; ++t) {                                              \
                T z = g[i * l + t] + tmp[i * l + t];                                       \
                g[i * l + t] = is_tanh ? TANH(z) : (T)0.5 * ((T)1 + TANH((T)0.5 * z));     \
            }                                                                              \
        }                                                                                  \
    }                                                                                      \
    ORC_CLONES void orc_sweep_out_fast_##SFX(int sru, const T *g0, const T *g1,            \
                                             const T *g2, const T *Xb, T *c, T *Hout,      \
                                             int64_t s, int64_t dh, int64_t l)             \
    {                                                                                      \
        _Pragma("omp parallel for schedule(static) if(dh * l > 2048)")                    \
        for (int64_t i = 0; i < dh; ++i) {                                                 \
            T ci = c[i];                                                                   \
            for (int64_t t = 0; t < l; ++t) {                                              \
                T f = g1[i * l + t];                                                       \
                ci = f * ci + ((T)1 - f) * g0[i * l + t];                                  \
                T h = g2[i * l + t] * TANH(ci);                                            \
                if (sru) h = h + ((T)1 - g2[i * l + t]) * Xb[i * l + t];                   \
                Hout[(s + t) * dh + i] = h;                                                \
            }                                                                              \
            c[i] = ci;                                                                     \
        }                                                                                  \
    }

FAST_ELEM(float, f32, tanhf)
FAST_ELEM(double, f64, tanh)
