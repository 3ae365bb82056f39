/*
 * TEST INFRASTRUCTURE ONLY -- the CPU oracle for the blocked SRU/QRNN path.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load this library.  The product path
 * (paper_1803_11389_b200) never links or calls it.
 *
 * A plain-C restatement of the reference algorithm in
 * /root/reference/pkg/src/rnnblock (rnnblock 0.1.0, pure Python + numba):
 *
 *   strict kernels  -- kernels.py:54-75  (_gemv_ref/_gemm_ref: ascending inner
 *                      index, one accumulator of the element type, no FMA
 *                      contraction: this file is compiled -ffp-contract=off)
 *   activations     -- kernels.py:236-241 (sigmoid(x) = 0.5*(1+tanh(0.5*x)))
 *   gate precompute -- blocked.py:123-150 (SRU 3 products + bias + sigmoid;
 *                      QRNN two taps, Xprev = [x_carry | Xb[:, :-1]])
 *   sweep           -- blocked.py:153-176 (c = f*c + (1-f)*cand, per lane)
 *   finalize        -- blocked.py:179-193 (QRNN o*tanh(c); SRU
 *                      r*tanh(c) + (1-r)*x)
 *   run_blocked     -- blocked.py:221-268 (layer-major, c and x_carry reset
 *                      to zero per layer, blocks from plan_blocks 38-50)
 *   stepwise oracle -- cells.py:167-228 (sru_step / qrnn_step /
 *                      run_layer_stepwise / run_stepwise)
 *   SplitMix64 + the top-24-bit uniform map -- kernels.py:253-305
 *
 * The "fast" GEMM (kernels.py:126-178) lives in oracle_fast.c.
 * Parity pin: tests/test_oracle_golden.py checks this file against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_SRU 1
#define ORC_QRNN 2
#define ORC_KERNEL_REFERENCE 0
#define ORC_KERNEL_FAST 1

/* oracle_fast.c */
void orc_gemm_fast_f32(const float *A, const float *Bt, float *C, int64_t m, int64_t k, int64_t n);
void orc_gemm_fast_f64(const double *A, const double *Bt, double *C, int64_t m, int64_t k, int64_t n);
void orc_set_threads(int n);
void orc_sig_bias_fast_f32(float *g, const float *b, int64_t dh, int64_t l);
void orc_sig_bias_fast_f64(double *g, const double *b, int64_t dh, int64_t l);
void orc_tap_act_fast_f32(float *g, const float *tmp, int64_t dh, int64_t l, int is_tanh);
void orc_tap_act_fast_f64(double *g, const double *tmp, int64_t dh, int64_t l, int is_tanh);
void orc_sweep_out_fast_f32(int sru, const float *g0, const float *g1, const float *g2, const float *Xb,
                            float *c, float *Hout, int64_t s, int64_t dh, int64_t l);
void orc_sweep_out_fast_f64(int sru, const double *g0, const double *g1, const double *g2, const double *Xb,
                            double *c, double *Hout, int64_t s, int64_t dh, int64_t l);

/* ---- SplitMix64 (kernels.py:253-289) and uniform map (292-305) ---- */
void orc_sm64_fill(uint64_t seed, uint64_t *out, int64_t n)
{
    uint64_t s = seed;
    for (int64_t i = 0; i < n; ++i) {
        s += 0x9E3779B97F4A7C15ULL;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        out[i] = z ^ (z >> 31);
    }
}

void orc_uniform(const uint64_t *raw, double *out, int64_t n)
{
    for (int64_t i = 0; i < n; ++i) {
        double u = (double)(raw[i] >> 40);
        out[i] = (u / 16777216.0) * 0.2 - 0.1;
    }
}

/* ---- type-generic body, instantiated for float and double ---- */
#define ORC_DEFINE(T, SFX, TANH)                                                           \
    static inline T sig_##SFX(T x) { return (T)0.5 * ((T)1.0 + TANH((T)0.5 * x)); }       \
                                                                                           \
    /* kernels.py:65-75: C[m x n] = A[m x k] . B[k x n], ascending p */                   \
    void orc_gemm_ref_##SFX(const T *A, const T *B, T *C, int64_t m, int64_t k, int64_t n) \
    {                                                                                      \
        for (int64_t i = 0; i < m; ++i)                                                    \
            for (int64_t j = 0; j < n; ++j) {                                              \
                T acc = (T)0;                                                              \
                for (int64_t p = 0; p < k; ++p) acc += A[i * k + p] * B[p * n + j];        \
                C[i * n + j] = acc;                                                        \
            }                                                                              \
    }                                                                                      \
                                                                                           \
    /* kernels.py:54-62 */                                                                 \
    void orc_gemv_ref_##SFX(const T *A, const T *x, T *y, int64_t m, int64_t k)           \
    {                                                                                      \
        for (int64_t i = 0; i < m; ++i) {                                                  \
            T acc = (T)0;                                                                  \
            for (int64_t j = 0; j < k; ++j) acc += A[i * k + j] * x[j];                    \
            y[i] = acc;                                                                    \
        }                                                                                  \
    }                                                                                      \
                                                                                           \
    /* gemm(kernel) dispatch, kernels.py:203-225; B given as [k x n]. The fast */          \
    /* kernel consumes B transposed (kernels.py:221). */                                   \
    static void gemm_##SFX(const T *A, const T *B, const T *Bt, T *C, int64_t m,          \
                           int64_t k, int64_t n, int kernel)                               \
    {                                                                                      \
        if (kernel == ORC_KERNEL_FAST)                                                     \
            orc_gemm_fast_##SFX(A, Bt, C, m, k, n);                                        \
        else                                                                               \
            orc_gemm_ref_##SFX(A, B, C, m, k, n);                                          \
    }                                                                                      \
                                                                                           \
    /* One layer, blocked (blocked.py:246-266).  Xin [L x din] row-major; Hout         */  \
    /* [L x dh].  mats: SRU {w_cand,w_forget,w_highway,b_forget,b_highway}; QRNN     */    \
    /* {w_cand,w_cand_prev,w_forget,w_forget_prev,w_out,w_out_prev} (model_io.py:29-33) */ \
    /* c_io / xc_io: optional carried state in and out (zero when NULL, as the         */  \
    /* reference's per-layer reset at blocked.py:247-248).                            */   \
    int orc_layer_blocked_##SFX(int kind, int64_t din, int64_t dh, const T *const *mats,  \
                                const T *Xin, int64_t L, int64_t Tb, int kernel, T *Hout,  \
                                T *c_io, T *xc_io)                                         \
    {                                                                                      \
        if (L < 1 || Tb < 1 || din < 1 || dh < 1) return -1;                               \
        if (kind == ORC_SRU && din != dh) return -1;                                       \
        int64_t nb = Tb < L ? Tb : L;                                                      \
        T *Xb = malloc(sizeof(T) * din * nb), *Xbt = malloc(sizeof(T) * din * nb);         \
        T *Xp = malloc(sizeof(T) * din * nb), *Xpt = malloc(sizeof(T) * din * nb);         \
        T *g0 = malloc(sizeof(T) * dh * nb), *g1 = malloc(sizeof(T) * dh * nb);            \
        T *g2 = malloc(sizeof(T) * dh * nb), *tmp = malloc(sizeof(T) * dh * nb);           \
        T *c = calloc(dh, sizeof(T)), *xc = calloc(din, sizeof(T));                        \
        if (c_io) memcpy(c, c_io, sizeof(T) * dh);                                         \
        if (xc_io && kind == ORC_QRNN) memcpy(xc, xc_io, sizeof(T) * din);                 \
        for (int64_t s = 0; s < L; s += Tb) {                                              \
            int64_t l = (L - s) < Tb ? (L - s) : Tb;                                       \
            /* Xb = layer_in[s:s+l].T (blocked.py:250); Xbt is its transpose */           \
            for (int64_t t = 0; t < l; ++t)                                                \
                for (int64_t i = 0; i < din; ++i) {                                        \
                    Xb[i * l + t] = Xin[(s + t) * din + i];                                \
                    Xbt[t * din + i] = Xin[(s + t) * din + i];                             \
                }                                                                          \
            if (kind == ORC_SRU) {                                                         \
                /* blocked.py:123-131 */                                                   \
                gemm_##SFX(mats[0], Xb, Xbt, g0, dh, din, l, kernel);                      \
                gemm_##SFX(mats[1], Xb, Xbt, g1, dh, din, l, kernel);                      \
                gemm_##SFX(mats[2], Xb, Xbt, g2, dh, din, l, kernel);                      \
                if (kernel == ORC_KERNEL_FAST) {                                           \
                    orc_sig_bias_fast_##SFX(g1, mats[3], dh, l);                           \
                    orc_sig_bias_fast_##SFX(g2, mats[4], dh, l);                           \
                } else                                                                     \
                for (int64_t i = 0; i < dh; ++i)                                           \
                    for (int64_t t = 0; t < l; ++t) {                                      \
                        g1[i * l + t] = sig_##SFX(g1[i * l + t] + mats[3][i]);             \
                        g2[i * l + t] = sig_##SFX(g2[i * l + t] + mats[4][i]);             \
                    }                                                                      \
            } else {                                                                       \
                /* blocked.py:134-150; Xprev = [x_carry | Xb[:, :-1]] (143) */            \
                for (int64_t i = 0; i < din; ++i) {                                        \
                    Xp[i * l] = xc[i];                                                     \
                    for (int64_t t = 1; t < l; ++t) Xp[i * l + t] = Xb[i * l + t - 1];     \
                }                                                                          \
                for (int64_t i = 0; i < din; ++i) {                                        \
                    Xpt[i] = xc[i];                                                        \
                    for (int64_t t = 1; t < l; ++t) Xpt[t * din + i] = Xbt[(t - 1) * din + i]; \
                }                                                                          \
                T *gs[3] = {g0, g1, g2};                                                   \
                for (int g = 0; g < 3; ++g) {                                              \
                    gemm_##SFX(mats[2 * g], Xb, Xbt, gs[g], dh, din, l, kernel);           \
                    gemm_##SFX(mats[2 * g + 1], Xp, Xpt, tmp, dh, din, l, kernel);         \
                    if (kernel == ORC_KERNEL_FAST) {                                       \
                        orc_tap_act_fast_##SFX(gs[g], tmp, dh, l, g == 0);                    \
                        continue;                                                          \
                    }                                                                      \
                    for (int64_t e = 0; e < dh * l; ++e) {                                 \
                        T z = gs[g][e] + tmp[e];                                           \
                        gs[g][e] = g == 0 ? TANH(z) : sig_##SFX(z);                        \
                    }                                                                      \
                }                                                                          \
                for (int64_t i = 0; i < din; ++i) xc[i] = Xb[i * l + l - 1];               \
            }                                                                              \
            /* sweep (blocked.py:153-162) then finalize (179-193) */                      \
            if (kernel == ORC_KERNEL_FAST) {                                               \
                orc_sweep_out_fast_##SFX(kind == ORC_SRU, g0, g1, g2, Xb, c, Hout, s, dh, l); \
                continue;                                                                  \
            }                                                                              \
            for (int64_t i = 0; i < dh; ++i) {                                             \
                T ci = c[i];                                                               \
                for (int64_t t = 0; t < l; ++t) {                                          \
                    T f = g1[i * l + t];                                                   \
                    ci = f * ci + ((T)1.0 - f) * g0[i * l + t];                            \
                    T th = TANH(ci);                                                       \
                    T o = g2[i * l + t];                                                   \
                    T h = o * th;                                                          \
                    if (kind == ORC_SRU) h = h + ((T)1.0 - o) * Xb[i * l + t];             \
                    Hout[(s + t) * dh + i] = h;                                            \
                }                                                                          \
                c[i] = ci;                                                                 \
            }                                                                              \
        }                                                                                  \
        if (c_io) memcpy(c_io, c, sizeof(T) * dh);                                         \
        if (xc_io && kind == ORC_QRNN) memcpy(xc_io, xc, sizeof(T) * din);                 \
        free(Xb); free(Xbt); free(Xp); free(Xpt); free(g0); free(g1); free(g2);           \
        free(tmp); free(c); free(xc);                                                      \
        return 0;                                                                          \
    }                                                                                      \
                                                                                           \
    /* One layer stepwise with the strict gemv (cells.py:167-214). */                     \
    int orc_layer_stepwise_##SFX(int kind, int64_t din, int64_t dh, const T *const *mats, \
                                 const T *Xin, int64_t L, T *Hout, T *c_io, T *xc_io)      \
    {                                                                                      \
        if (L < 1 || din < 1 || dh < 1) return -1;                                         \
        if (kind == ORC_SRU && din != dh) return -1;                                       \
        T *c = calloc(dh, sizeof(T)), *xp = calloc(din, sizeof(T));                        \
        T *a = malloc(sizeof(T) * dh), *b = malloc(sizeof(T) * dh);                        \
        T *f = malloc(sizeof(T) * dh), *o = malloc(sizeof(T) * dh);                        \
        T *cand = malloc(sizeof(T) * dh);                                                  \
        if (c_io) memcpy(c, c_io, sizeof(T) * dh);                                         \
        if (xc_io && kind == ORC_QRNN) memcpy(xp, xc_io, sizeof(T) * din);                 \
        for (int64_t t = 0; t < L; ++t) {                                                  \
            const T *x = Xin + t * din;                                                    \
            if (kind == ORC_SRU) {                                                         \
                orc_gemv_ref_##SFX(mats[0], x, cand, dh, din);                             \
                orc_gemv_ref_##SFX(mats[1], x, a, dh, din);                                \
                orc_gemv_ref_##SFX(mats[2], x, b, dh, din);                                \
                for (int64_t i = 0; i < dh; ++i) {                                         \
                    f[i] = sig_##SFX(a[i] + mats[3][i]);                                   \
                    o[i] = sig_##SFX(b[i] + mats[4][i]);                                   \
                }                                                                          \
            } else {                                                                       \
                T *dst[3] = {cand, f, o};                                                  \
                for (int g = 0; g < 3; ++g) {                                              \
                    orc_gemv_ref_##SFX(mats[2 * g], x, a, dh, din);                        \
                    orc_gemv_ref_##SFX(mats[2 * g + 1], xp, b, dh, din);                   \
                    for (int64_t i = 0; i < dh; ++i) {                                     \
                        T z = a[i] + b[i];                                                 \
                        dst[g][i] = g == 0 ? TANH(z) : sig_##SFX(z);                       \
                    }                                                                      \
                }                                                                          \
            }                                                                              \
            for (int64_t i = 0; i < dh; ++i) {                                             \
                c[i] = f[i] * c[i] + ((T)1.0 - f[i]) * cand[i];                            \
                T h = o[i] * TANH(c[i]);                                                   \
                if (kind == ORC_SRU) h = h + ((T)1.0 - o[i]) * x[i];                       \
                Hout[t * dh + i] = h;                                                      \
            }                                                                              \
            memcpy(xp, x, sizeof(T) * din);                                                \
        }                                                                                  \
        if (c_io) memcpy(c_io, c, sizeof(T) * dh);                                         \
        if (xc_io && kind == ORC_QRNN) memcpy(xc_io, xp, sizeof(T) * din);                 \
        free(c); free(xp); free(a); free(b); free(f); free(o); free(cand);                 \
        return 0;                                                                          \
    }

ORC_DEFINE(float, f32, tanhf)
ORC_DEFINE(double, f64, tanh)

/* ---- LSTM, instantiated for float and double ----
 * mats (cells.py:46-58, model_io.py:29-33): w_forget, w_input, w_output,
 * w_cand [dh x din], u_forget, u_input, u_output, u_cand [dh x dh],
 * b_forget, b_input, b_output, b_cand [dh].  Gate slot g: 0 f, 1 i, 2 o, 3 c.
 * c_io / h_io: optional state in and out (zero when NULL, as the
 * reference's h = c = 0 at blocked.py:284-285 / cells.py:138-143). */
#define ORC_DEFINE_LSTM(T, SFX, TANH)                                                      \
    /* lstm_run_precomputed, blocked.py:271-305: per block the four W Xb products +   */  \
    /* bias ((W x) + b), then per step pre = that + U h_{t-1} (strict gemv order).     */  \
    int orc_lstm_blocked_##SFX(int64_t din, int64_t dh, const T *const *mats, const T *Xin, \
                               int64_t L, int64_t Tb, int kernel, T *Hout, T *c_io, T *h_io) \
    {                                                                                      \
        if (L < 1 || Tb < 1 || din < 1 || dh < 1) return -1;                               \
        int64_t nb = Tb < L ? Tb : L;                                                      \
        T *Xb = malloc(sizeof(T) * din * nb), *Xbt = malloc(sizeof(T) * din * nb);         \
        T *g[4];                                                                           \
        for (int q = 0; q < 4; ++q) g[q] = malloc(sizeof(T) * dh * nb);                    \
        T *u = malloc(sizeof(T) * dh), *act = malloc(sizeof(T) * 4 * dh);                  \
        T *c = calloc(dh, sizeof(T)), *h = calloc(dh, sizeof(T));                          \
        if (c_io) memcpy(c, c_io, sizeof(T) * dh);                                         \
        if (h_io) memcpy(h, h_io, sizeof(T) * dh);                                         \
        for (int64_t s = 0; s < L; s += Tb) {                                              \
            int64_t l = (L - s) < Tb ? (L - s) : Tb;                                       \
            for (int64_t t = 0; t < l; ++t)                                                \
                for (int64_t i = 0; i < din; ++i) {                                        \
                    Xb[i * l + t] = Xin[(s + t) * din + i];                                \
                    Xbt[t * din + i] = Xin[(s + t) * din + i];                             \
                }                                                                          \
            for (int q = 0; q < 4; ++q) {                                                  \
                gemm_##SFX(mats[q], Xb, Xbt, g[q], dh, din, l, kernel);                    \
                for (int64_t i = 0; i < dh; ++i)                                           \
                    for (int64_t t = 0; t < l; ++t) g[q][i * l + t] += mats[8 + q][i];     \
            }                                                                              \
            for (int64_t t = 0; t < l; ++t) {                                              \
                for (int q = 0; q < 4; ++q) {                                              \
                    orc_gemv_ref_##SFX(mats[4 + q], h, u, dh, dh);                         \
                    for (int64_t i = 0; i < dh; ++i) {                                     \
                        T z = g[q][i * l + t] + u[i];                                      \
                        act[q * dh + i] = q == 3 ? TANH(z) : sig_##SFX(z);                 \
                    }                                                                      \
                }                                                                          \
                for (int64_t i = 0; i < dh; ++i) {                                         \
                    c[i] = act[i] * c[i] + act[dh + i] * act[3 * dh + i];                  \
                    h[i] = act[2 * dh + i] * TANH(c[i]);                                   \
                    Hout[(s + t) * dh + i] = h[i];                                         \
                }                                                                          \
            }                                                                              \
        }                                                                                  \
        if (c_io) memcpy(c_io, c, sizeof(T) * dh);                                         \
        if (h_io) memcpy(h_io, h, sizeof(T) * dh);                                         \
        free(Xb); free(Xbt); free(u); free(act); free(c); free(h);                         \
        for (int q = 0; q < 4; ++q) free(g[q]);                                            \
        return 0;                                                                          \
    }                                                                                      \
                                                                                           \
    /* lstm_step, cells.py:153-164: sigma(W x + U h + b) per gate, strict gemv. */         \
    int orc_lstm_stepwise_##SFX(int64_t din, int64_t dh, const T *const *mats, const T *Xin, \
                                int64_t L, T *Hout, T *c_io, T *h_io)                      \
    {                                                                                      \
        if (L < 1 || din < 1 || dh < 1) return -1;                                         \
        T *a = malloc(sizeof(T) * dh), *b = malloc(sizeof(T) * dh);                        \
        T *act = malloc(sizeof(T) * 4 * dh);                                               \
        T *c = calloc(dh, sizeof(T)), *h = calloc(dh, sizeof(T));                          \
        if (c_io) memcpy(c, c_io, sizeof(T) * dh);                                         \
        if (h_io) memcpy(h, h_io, sizeof(T) * dh);                                         \
        for (int64_t t = 0; t < L; ++t) {                                                  \
            const T *x = Xin + t * din;                                                    \
            for (int q = 0; q < 4; ++q) {                                                  \
                orc_gemv_ref_##SFX(mats[q], x, a, dh, din);                                \
                orc_gemv_ref_##SFX(mats[4 + q], h, b, dh, dh);                             \
                for (int64_t i = 0; i < dh; ++i) {                                         \
                    T z = a[i] + b[i] + mats[8 + q][i];                                    \
                    act[q * dh + i] = q == 3 ? TANH(z) : sig_##SFX(z);                     \
                }                                                                          \
            }                                                                              \
            for (int64_t i = 0; i < dh; ++i) {                                             \
                c[i] = act[i] * c[i] + act[dh + i] * act[3 * dh + i];                      \
                h[i] = act[2 * dh + i] * TANH(c[i]);                                       \
                Hout[t * dh + i] = h[i];                                                   \
            }                                                                              \
        }                                                                                  \
        if (c_io) memcpy(c_io, c, sizeof(T) * dh);                                         \
        if (h_io) memcpy(h_io, h, sizeof(T) * dh);                                         \
        free(a); free(b); free(act); free(c); free(h);                                     \
        return 0;                                                                          \
    }

ORC_DEFINE_LSTM(float, f32, tanhf)
ORC_DEFINE_LSTM(double, f64, tanh)
