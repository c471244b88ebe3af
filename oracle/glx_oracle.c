/*
 * glx_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference glycemlp hot path
 * (/root/reference/pkg/src/glycemlp/kernels.py), used as the parity checker
 * for the CUDA path and as the CPU baseline in bench.py. Nothing in the
 * product path (paper_1908_07847_b200/) links, loads or calls this file.
 *
 * Numerics follow the reference exactly:
 *   - every dot product accumulates in float64 over fixed 16-wide blocks,
 *     blocks combined in index order, bias added last   (kernels.py:102-122)
 *   - sigmoid = f32(1 / (1 + exp(-z))) in float64 with glibc exp, which is
 *     what numba's llvm.exp.f64 lowers to                  (kernels.py:118-122)
 *   - delta = (err * a) * (1 - a), left to right           (kernels.py:125-129)
 *   - update w = f32(f64(w) - step * f64(x)), unfused     (kernels.py:132-139)
 * Build with -ffp-contract=off (see oracle/Makefile): no FMA contraction, so
 * every float64 op is a separately rounded IEEE op as in the numba code.
 *
 * Parity pin: tests/test_oracle.py checks these functions byte-for-byte
 * against fixtures produced by the reference itself (tests/golden/make_golden.py).
 *
 * Extensions beyond the reference, needed
 * for the batch and K>1 configurations the reference cannot run:
 *   - orc_train_batch: B-row mini/full-batch gradient descent restated from
 *     kernels.py:264-295; B=1 reproduces
 *     train_segment_seq bit-for-bit (asserted in tests/test_oracle.py).
 *   - K sigmoid outputs with one-hot targets, argmax prediction (lowest index
 *     wins ties); K=1 keeps the reference's o >= 0.5f rule.
 *   - loss = sum over rows of 0.5*(t-o)^2 (network.py:186 per-row error).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdatomic.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_BLOCK 16 /* kernels.py:31 */

/* kernels.py:102-115 _blocked_dot */
static inline double blocked_dot(const float *w, const float *x, int n) {
    double acc = 0.0;
    for (int b0 = 0; b0 < n; b0 += ORC_BLOCK) {
        int b1 = b0 + ORC_BLOCK < n ? b0 + ORC_BLOCK : n;
        double part = 0.0;
        for (int i = b0; i < b1; i++) part += (double)w[i] * (double)x[i];
        acc += part;
    }
    return acc;
}

/* kernels.py:118-122 _activation: sigmoid(blocked dot + bias) rounded to f32 */
static inline float activation(const float *wrow, const float *x, int n) {
    double z = blocked_dot(wrow, x, n) + (double)wrow[n];
    return (float)(1.0 / (1.0 + exp(-z)));
}

/* kernels.py:125-129 _delta_from_error */
static inline double delta_from_error(double err, float act) {
    double a = (double)act;
    return err * a * (1.0 - a);
}

/* kernels.py:132-139 _update_row */
static inline void update_row(float *wrow, const float *x, int n, double step) {
    for (int i = 0; i < n; i++) wrow[i] = (float)((double)wrow[i] - step * (double)x[i]);
    wrow[n] = (float)((double)wrow[n] - step);
}

double orc_sigmoid64(double x) { return 1.0 / (1.0 + exp(-x)); } /* kernels.py:142-145 */

/* Forward pass of one row (network.py:128-135): hidden[H], out[K]. */
void orc_forward_row(const float *w_ih, const float *w_ho, const float *x,
                     int D, int H, int K, float *hidden, float *out) {
    for (int j = 0; j < H; j++) hidden[j] = activation(w_ih + (int64_t)j * (D + 1), x, D);
    for (int k = 0; k < K; k++) out[k] = activation(w_ho + (int64_t)k * (H + 1), hidden, H);
}

/* kernels.py:264-295 train_segment_seq: per-instance online SGD, in place. */
int orc_train_online_seq(float *w_ih, float *w_ho, const float *feats, const float *targets,
                         int64_t rows, int D, int H, int64_t epochs, double lr) {
    float *h = (float *)malloc(sizeof(float) * (size_t)H);
    if (!h) return -1;
    for (int64_t e = 0; e < epochs; e++) {
        for (int64_t r = 0; r < rows; r++) {
            const float *x = feats + r * D;
            for (int j = 0; j < H; j++) h[j] = activation(w_ih + (int64_t)j * (D + 1), x, D);
            /* output: 16-blocked partials over h, bias as the last partial (:277-287) */
            float o = activation(w_ho, h, H);
            double d_o = delta_from_error((double)o - (double)targets[r], o);
            double step_o = lr * d_o;
            for (int j = 0; j < H; j++) { /* hidden first, from the pre-update w_ho (:290-292) */
                double d_h = delta_from_error((double)w_ho[j] * d_o, h[j]);
                update_row(w_ih + (int64_t)j * (D + 1), x, D, lr * d_h);
            }
            for (int j = 0; j < H; j++) w_ho[j] = (float)((double)w_ho[j] - step_o * (double)h[j]);
            w_ho[H] = (float)((double)w_ho[H] - step_o);
        }
    }
    free(h);
    return 0;
}

/* ---------------------------------------------------------------------------
 * kernels.py:298-349 train_segment_par + kernels.py:83-95 _barrier:
 * the neuron-parallel engine. Worker w owns BLOCK-aligned hidden slices
 * (kernels.py:317-321), publishes its output-dot partials, meets the others
 * at a centralised generation spin barrier, recombines all partials
 * redundantly, updates its own slice and meets again. Bit-identical to seq.
 * ------------------------------------------------------------------------- */
typedef struct { _Atomic int64_t cnt; _Atomic int64_t gen; char pad[48]; } orc_sync_t;

static inline void spin_barrier(orc_sync_t *s, int nw) {
    int64_t my_gen = atomic_load_explicit(&s->gen, memory_order_acquire);
    if (atomic_fetch_add_explicit(&s->cnt, 1, memory_order_acq_rel) == nw - 1) {
        atomic_store_explicit(&s->cnt, 0, memory_order_release);
        atomic_store_explicit(&s->gen, my_gen + 1, memory_order_release);
    } else {
        while (atomic_load_explicit(&s->gen, memory_order_acquire) == my_gen) { }
    }
}

int orc_train_online_par(float *w_ih, float *w_ho, const float *feats, const float *targets,
                         int64_t rows, int D, int H, int64_t epochs, double lr, int nw) {
    int nb = (H + ORC_BLOCK - 1) / ORC_BLOCK;
    if (nw < 1) nw = 1;
    float *h = (float *)malloc(sizeof(float) * (size_t)H);
    double *part = (double *)malloc(sizeof(double) * (size_t)(nb + 1));
    orc_sync_t *sync = (orc_sync_t *)aligned_alloc(64, sizeof(orc_sync_t));
    if (!h || !part || !sync) { free(h); free(part); free(sync); return -1; }
    atomic_init(&sync->cnt, 0);
    atomic_init(&sync->gen, 0);
#ifdef _OPENMP
#pragma omp parallel num_threads(nw)
#endif
    {
#ifdef _OPENMP
        int w = omp_get_thread_num();
        int nwr = omp_get_num_threads();
#else
        int w = 0, nwr = 1;
#endif
        int j_lo = (w * nb / nwr) * ORC_BLOCK;
        int j_hi = ((w + 1) * nb / nwr) * ORC_BLOCK; if (j_hi > H) j_hi = H;
        int b_lo = w * nb / nwr, b_hi = (w + 1) * nb / nwr;
        for (int64_t e = 0; e < epochs; e++) {
            for (int64_t r = 0; r < rows; r++) {
                const float *x = feats + r * D;
                for (int j = j_lo; j < j_hi; j++) h[j] = activation(w_ih + (int64_t)j * (D + 1), x, D);
                for (int b = b_lo; b < b_hi; b++) {
                    int j1 = (b + 1) * ORC_BLOCK < H ? (b + 1) * ORC_BLOCK : H;
                    double p = 0.0;
                    for (int j = b * ORC_BLOCK; j < j1; j++) p += (double)w_ho[j] * (double)h[j];
                    part[b] = p;
                }
                if (w == 0) part[nb] = (double)w_ho[H];
                spin_barrier(sync, nwr);
                double z = 0.0;
                for (int b = 0; b <= nb; b++) z += part[b];
                float o = (float)(1.0 / (1.0 + exp(-z)));
                double d_o = delta_from_error((double)o - (double)targets[r], o);
                double step_o = lr * d_o;
                for (int j = j_lo; j < j_hi; j++) {
                    double d_h = delta_from_error((double)w_ho[j] * d_o, h[j]);
                    update_row(w_ih + (int64_t)j * (D + 1), x, D, lr * d_h);
                }
                for (int j = j_lo; j < j_hi; j++) w_ho[j] = (float)((double)w_ho[j] - step_o * (double)h[j]);
                if (w == 0) w_ho[H] = (float)((double)w_ho[H] - step_o);
                spin_barrier(sync, nwr);
            }
        }
    }
    free(h); free(part); free(sync);
    return 0;
}

/* ---------------------------------------------------------------------------
 * Batch restatement (no reference code exists).
 * Per batch of B rows, every row's forward/delta uses the batch-start
 * weights; per-row step s = (lr/B)*delta in f64; dW accumulates s*[x,1] in
 * f64 in row order; W <- f32(f64(W) - dW) once per batch. With B=1 this is
 * exactly _update_row's association, hence bit-identical to
 * orc_train_online_seq (the anchor test). K outputs: targets T is rows x K.
 * ------------------------------------------------------------------------- */
int orc_train_batch(float *w_ih, float *w_ho, const float *feats, const float *T,
                    int64_t rows, int D, int H, int K, int64_t epochs, int64_t B, double lr) {
    if (B < 1) B = 1;
    const int64_t P1 = (int64_t)H * (D + 1), P2 = (int64_t)K * (H + 1);
    double *dW1 = (double *)malloc(sizeof(double) * (size_t)P1);
    double *dW2 = (double *)malloc(sizeof(double) * (size_t)P2);
    float *h = (float *)malloc(sizeof(float) * (size_t)H);
    float *o = (float *)malloc(sizeof(float) * (size_t)K);
    double *d_o = (double *)malloc(sizeof(double) * (size_t)K);
    if (!dW1 || !dW2 || !h || !o || !d_o) { free(dW1); free(dW2); free(h); free(o); free(d_o); return -1; }
    const double scale = lr / (double)B;
    for (int64_t e = 0; e < epochs; e++) {
        for (int64_t b0 = 0; b0 < rows; b0 += B) {
            int64_t b1 = b0 + B < rows ? b0 + B : rows;
            memset(dW1, 0, sizeof(double) * (size_t)P1);
            memset(dW2, 0, sizeof(double) * (size_t)P2);
            for (int64_t r = b0; r < b1; r++) {
                const float *x = feats + r * D;
                orc_forward_row(w_ih, w_ho, x, D, H, K, h, o);
                for (int k = 0; k < K; k++)
                    d_o[k] = delta_from_error((double)o[k] - (double)T[r * K + k], o[k]);
                for (int j = 0; j < H; j++) {
                    double err;
                    if (K == 1) err = (double)w_ho[j] * d_o[0];
                    else { err = 0.0; for (int k = 0; k < K; k++) err += (double)w_ho[(int64_t)k * (H + 1) + j] * d_o[k]; }
                    double s = scale * delta_from_error(err, h[j]);
                    double *g = dW1 + (int64_t)j * (D + 1);
                    for (int i = 0; i < D; i++) g[i] += s * (double)x[i];
                    g[D] += s;
                }
                for (int k = 0; k < K; k++) {
                    double s = scale * d_o[k];
                    double *g = dW2 + (int64_t)k * (H + 1);
                    for (int j = 0; j < H; j++) g[j] += s * (double)h[j];
                    g[H] += s;
                }
            }
            for (int64_t p = 0; p < P1; p++) w_ih[p] = (float)((double)w_ih[p] - dW1[p]);
            for (int64_t p = 0; p < P2; p++) w_ho[p] = (float)((double)w_ho[p] - dW2[p]);
        }
    }
    free(dW1); free(dW2); free(h); free(o); free(d_o);
    return 0;
}

/* Row-parallel full-batch epoch (B = rows) for the CPU baseline: per-thread
 * f64 partial gradients over contiguous row ranges, combined in thread
 * order. Same math as orc_train_batch(B=rows) up to f64 summation order. */
int orc_train_batch_par(float *w_ih, float *w_ho, const float *feats, const float *T,
                        int64_t rows, int D, int H, int K, int64_t epochs, double lr, int nw) {
    if (nw < 1) nw = 1;
    const int64_t P1 = (int64_t)H * (D + 1), P2 = (int64_t)K * (H + 1), P = P1 + P2;
    double *acc = (double *)calloc((size_t)nw * (size_t)P, sizeof(double));
    if (!acc) return -1;
    const double scale = lr / (double)rows;
    for (int64_t e = 0; e < epochs; e++) {
        memset(acc, 0, sizeof(double) * (size_t)nw * (size_t)P);
#ifdef _OPENMP
#pragma omp parallel num_threads(nw)
#endif
        {
#ifdef _OPENMP
            int w = omp_get_thread_num();
            int nwr = omp_get_num_threads();
#else
            int w = 0, nwr = 1;
#endif
            float *h = (float *)malloc(sizeof(float) * (size_t)H);
            float *o = (float *)malloc(sizeof(float) * (size_t)K);
            double *d_o = (double *)malloc(sizeof(double) * (size_t)K);
            double *g1 = acc + (int64_t)w * P, *g2 = g1 + P1;
            int64_t r0 = rows * w / nwr, r1 = rows * (w + 1) / nwr;
            for (int64_t r = r0; r < r1; r++) {
                const float *x = feats + r * D;
                orc_forward_row(w_ih, w_ho, x, D, H, K, h, o);
                for (int k = 0; k < K; k++)
                    d_o[k] = delta_from_error((double)o[k] - (double)T[r * K + k], o[k]);
                for (int j = 0; j < H; j++) {
                    double err = 0.0;
                    for (int k = 0; k < K; k++) err += (double)w_ho[(int64_t)k * (H + 1) + j] * d_o[k];
                    double s = scale * delta_from_error(err, h[j]);
                    double *g = g1 + (int64_t)j * (D + 1);
                    for (int i = 0; i < D; i++) g[i] += s * (double)x[i];
                    g[D] += s;
                }
                for (int k = 0; k < K; k++) {
                    double s = scale * d_o[k];
                    double *g = g2 + (int64_t)k * (H + 1);
                    for (int j = 0; j < H; j++) g[j] += s * (double)h[j];
                    g[H] += s;
                }
            }
            free(h); free(o); free(d_o);
        }
        for (int64_t p = 0; p < P; p++) {
            double s = 0.0;
            for (int w = 0; w < nw; w++) s += acc[(int64_t)w * P + p];
            if (p < P1) w_ih[p] = (float)((double)w_ih[p] - s);
            else w_ho[p - P1] = (float)((double)w_ho[p - P1] - s);
        }
    }
    free(acc);
    return 0;
}

/* One epoch's gradient SUM at fixed weights (the quantity glx_batch_grad
 * returns): grad = [sum_r dh_r (x) [x_r, 1] (H(D+1)) | sum_r d_o,r (x) [h_r, 1]
 * (K(H+1)) | loss | tp tn fp fn], deltas as in orc_train_batch with lr/B = 1
 * (kernels.py:125-129 op order), rows split over nw OpenMP threads, f64
 * partials combined in thread order. K == 1 counts as in orc_eval. */
int orc_batch_grad_par(const float *w_ih, const float *w_ho, const float *feats, const float *T,
                       int64_t rows, int D, int H, int K, double *grad, int nw) {
    if (nw < 1) nw = 1;
    const int64_t P1 = (int64_t)H * (D + 1), P2 = (int64_t)K * (H + 1), P = P1 + P2 + 5;
    double *acc = (double *)calloc((size_t)nw * (size_t)P, sizeof(double));
    if (!acc) return -1;
#ifdef _OPENMP
#pragma omp parallel num_threads(nw)
#endif
    {
#ifdef _OPENMP
        int w = omp_get_thread_num();
        int nwr = omp_get_num_threads();
#else
        int w = 0, nwr = 1;
#endif
        float *h = (float *)malloc(sizeof(float) * (size_t)H);
        float *o = (float *)malloc(sizeof(float) * (size_t)K);
        double *d_o = (double *)malloc(sizeof(double) * (size_t)K);
        double *g1 = acc + (int64_t)w * P, *g2 = g1 + P1, *st = g2 + P2;
        int64_t r0 = rows * w / nwr, r1 = rows * (w + 1) / nwr;
        for (int64_t r = r0; r < r1; r++) {
            const float *x = feats + r * D;
            orc_forward_row(w_ih, w_ho, x, D, H, K, h, o);
            for (int k = 0; k < K; k++) {
                d_o[k] = delta_from_error((double)o[k] - (double)T[r * K + k], o[k]);
                double e = (double)T[r * K + k] - (double)o[k];
                st[0] += 0.5 * e * e;
            }
            if (K == 1) {
                int pred = o[0] >= 0.5f, pos = T[r] >= 0.5f;
                st[pred && pos ? 1 : !pred && !pos ? 2 : pred ? 3 : 4] += 1.0;
            }
            for (int j = 0; j < H; j++) {
                double err = 0.0;
                for (int k = 0; k < K; k++) err += (double)w_ho[(int64_t)k * (H + 1) + j] * d_o[k];
                double s = delta_from_error(err, h[j]);
                double *g = g1 + (int64_t)j * (D + 1);
                for (int i = 0; i < D; i++) g[i] += s * (double)x[i];
                g[D] += s;
            }
            for (int k = 0; k < K; k++) {
                double *g = g2 + (int64_t)k * (H + 1);
                for (int j = 0; j < H; j++) g[j] += d_o[k] * (double)h[j];
                g[H] += d_o[k];
            }
        }
        free(h); free(o); free(d_o);
    }
    for (int64_t p = 0; p < P; p++) {
        double s = 0.0;
        for (int w = 0; w < nw; w++) s += acc[(int64_t)w * P + p];
        grad[p] = s;
    }
    free(acc);
    return 0;
}

/* kernels.py:352-375 eval_counts, plus the K>1 and loss extensions.
 * K == 1: counts = (tp, tn, fp, fn), poor (label 1) positive, pred = o >= 0.5f.
 * K  > 1: counts = (correct, wrong, 0, 0), pred = argmax (lowest index on ties).
 * loss_sum = sum over rows and outputs of 0.5*(t - o)^2 in f64. */
void orc_eval(const float *w_ih, const float *w_ho, const float *feats, const uint8_t *labels,
              int64_t rows, int D, int H, int K, int64_t *counts, double *loss_sum) {
    float *h = (float *)malloc(sizeof(float) * (size_t)H);
    float *o = (float *)malloc(sizeof(float) * (size_t)K);
    int64_t tp = 0, tn = 0, fp = 0, fn = 0;
    double loss = 0.0;
    for (int64_t r = 0; r < rows; r++) {
        orc_forward_row(w_ih, w_ho, feats + r * D, D, H, K, h, o);
        if (K == 1) {
            int pred = o[0] >= 0.5f ? 1 : 0;
            if (pred == 1) { if (labels[r] == 1) tp++; else fp++; }
            else { if (labels[r] == 1) fn++; else tn++; }
            double d = (double)labels[r] - (double)o[0];
            loss += 0.5 * d * d;
        } else {
            int best = 0;
            for (int k = 1; k < K; k++) if (o[k] > o[best]) best = k;
            if (best == (int)labels[r]) tp++; else tn++;
            for (int k = 0; k < K; k++) {
                double d = (labels[r] == k ? 1.0 : 0.0) - (double)o[k];
                loss += 0.5 * d * d;
            }
        }
    }
    if (K == 1) { counts[0] = tp; counts[1] = tn; counts[2] = fp; counts[3] = fn; }
    else { counts[0] = tp; counts[1] = tn; counts[2] = 0; counts[3] = 0; }
    if (loss_sum) *loss_sum = loss;
    free(h); free(o);
}

/* Sweep baseline: n_nets independent online networks on one dataset, one
 * network per OpenMP thread (dynamic schedule). Weights are packed per
 * network at w_off[n] as [w_ih (H(D+1)) | w_ho (H+1)]. */
int orc_train_sweep(int64_t n_nets, const int32_t *H_per_net, const int64_t *w_off, float *w_pool,
                    const float *feats, const float *targets, int64_t rows, int D,
                    int64_t epochs, double lr, int nw) {
    int rc = 0;
#ifdef _OPENMP
#pragma omp parallel for schedule(dynamic, 1) num_threads(nw) reduction(|:rc)
#endif
    for (int64_t n = 0; n < n_nets; n++) {
        int H = H_per_net[n];
        float *w_ih = w_pool + w_off[n];
        float *w_ho = w_ih + (int64_t)H * (D + 1);
        rc |= orc_train_online_seq(w_ih, w_ho, feats, targets, rows, D, H, epochs, lr);
    }
    return rc;
}

int orc_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
