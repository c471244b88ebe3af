// glx_kernels.h -- internal launch descriptors shared by the .cu files and the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>

namespace glx {

// --------------------------------------------------------------- online SGD
struct OnlineNetDesc {
    float* w_ih;      // H x (D+1), reference layout (network.py:84-90)
    float* w_ho;      // H + 1
    int H;
    int warp0;        // first warp of this network inside its CTA
    int nwarps;
    int bar_id;       // named barrier id (1..15)
    int scratch_off;  // byte offset of this network's scratch in dynamic smem
    int pad;
};

struct OnlineLaunch {
    const OnlineNetDesc* nets;  // device
    const int2* cta_nets;       // device: (first net, count) per CTA
    int n_ctas;
    int threads;
    size_t smem_bytes;
    bool x_in_smem;
    bool ref64;
    int mt;  // fp32 hidden units per thread (1, 2 or 4)
    bool one_warp = false;  // every network fits one warp (fp32 MT kernel fast path)
    const float* X;  // device, (N, D)
    const float* T;  // device, (N,)
    int64_t N;
    int D;
    int64_t epochs;
    double lr;
};

int online_dp_for(int D);
// ref64 online SGD of one network with H <= 64 and input_dim <= 33 (f64-resident rows)
size_t online_ref64_small_smem(int64_t N, int D);
cudaError_t launch_online_ref64_small(float* w_ih, float* w_ho, int H, const float* X, const float* T, int64_t N,
                                      int D, int64_t epochs, double lr, cudaStream_t st);
cudaError_t launch_online(const OnlineLaunch& L, cudaStream_t st);
size_t online_scratch_bytes(int H, bool ref64);

// -------------------------------------------------------------- batch epoch
struct BatchGeom {
    int D, H, DP, LD, MT, TPG, G, R, RPG, HP;
    int64_t N, ntiles;
    int grid;
    int P1;   // H*(D+1)
    int PS;   // per-CTA partial record stride (floats)
    int WKS;  // kernel weight-copy stride (floats)
    size_t smem;
    // three-role kernel (glx_batch3.cu) only
    int UA, QR, AG;
    int off_dob, off_opart, off_z, off_x;
};
using Batch3Geom = BatchGeom;

// kernel weight copy layout (floats): W1s[H][DP] (scaled by -log2 e, bias at
// slot D, zero beyond), w2s[H] (scaled), b2s (scaled), w2r[H] (raw)
inline int wk_w2s(const BatchGeom& g) { return g.H * g.DP; }
inline int wk_b2s(const BatchGeom& g) { return g.H * g.DP + g.H; }
inline int wk_w2r(const BatchGeom& g) { return g.H * g.DP + g.H + 1; }

// per-CTA partial record: [dW1acc (P1) | dW2acc (H) | dsum | loss | c0 c1 c2 c3]
inline int ps_acc2(const BatchGeom& g) { return g.P1; }
inline int ps_dsum(const BatchGeom& g) { return g.P1 + g.H; }
inline int ps_loss(const BatchGeom& g) { return g.P1 + g.H + 1; }
inline int ps_cnt(const BatchGeom& g) { return g.P1 + g.H + 2; }

bool batch_geometry(int64_t N, int D, int H, int n_sms, bool train, BatchGeom* g);
// col_min/col_max (optional): min-max normalise the features while packing
cudaError_t launch_pack_rows(const float* X, const float* T, const uint8_t* labels, int64_t N, int D, int LD,
                             float* Xp, cudaStream_t st, const float* col_min = nullptr,
                             const float* col_max = nullptr);
// TMA-staged packing (glx_data.cu), used by launch_pack_rows when aligned
bool pack_tiled_ok(const void* X, const void* T, const void* labels, const void* Xp, int D, int LD);
cudaError_t launch_pack_tiled(const float* X, const float* T, const uint8_t* labels, int64_t N, int D, int LD,
                              const float* col_min, const float* col_max, float* Xp, cudaStream_t st);
// min-max normalisation (glx_data.cu); work = 2*D ints
cudaError_t launch_minmax_fit(const float* X, int64_t N, int D, int* work, float* col_min, float* col_max,
                              cudaStream_t st);
cudaError_t launch_minmax_apply(const float* X, int64_t N, int D, const float* col_min, const float* col_max,
                                float* Y, cudaStream_t st);
cudaError_t launch_batch_prep(const BatchGeom& g, const float* W1, const float* W2, float* Wk0, float* Wk1,
                              cudaStream_t st);
cudaError_t launch_batch_epoch(const BatchGeom& g, const float* Xp, const float* Wk, float* part, bool train,
                               cudaStream_t st);
// reduce the per-CTA partials; if train, apply the SGD update to W1/W2 and
// write the next kernel weight copy. stats (may be null): [loss, c0, c1, c2, c3]
cudaError_t launch_batch_dp_update(const BatchGeom& g, float* W1, float* W2, float* Wk_next, const double* grad,
                                   double lr_over_n, double* stats_slot, int* nonfinite, cudaStream_t st);
cudaError_t launch_batch_update(const BatchGeom& g, const float* part, float* W1, float* W2, const float* Wk_cur,
                                float* Wk_next, double lr_over_n, bool train, double* stats, int* nonfinite,
                                cudaStream_t st);

#ifndef GLX3_TILE_ROWS
#define GLX3_TILE_ROWS 256
#endif
// three-role (forward / activation / backward) epoch kernel; same partial record
bool batch3_geometry(int64_t N, int D, int H, int n_sms, Batch3Geom* g);
cudaError_t launch_batch3_epoch(const Batch3Geom& g, const float* Xp, const float* Wk, float* part, cudaStream_t st);
// tcgen05 epoch kernel (glx_batchtc.cu): H = 128 or 256, D <= 33; same partial record as batch3
bool batchtc_geometry(int64_t N, int D, int H, int n_sms, BatchGeom* g);
int pick_dp(int D);  // glx_batch.cu: weight-row stride of the FP32 batch kernels (-1: D too wide)
// the tcgen05 epoch kernel reads the rows pre-laid-out per 64-row tile (tf32 MMA
// operands): batchtc_tile_bytes of scratch filled once per training call from the
// packed rows by launch_batchtc_pack
size_t batchtc_tile_bytes(const BatchGeom& g);
cudaError_t launch_batchtc_pack(const BatchGeom& g, const float* Xp, void* tiles, cudaStream_t st);
cudaError_t launch_batchtc_epoch(const BatchGeom& g, const void* tiles, const float* Wk, float* part, cudaStream_t st,
                                 int* dbg = nullptr);
// ints of the tcgen05 kernels' pipeline-checker buffer (debug runs; glx_batchtc.cu)
size_t pipeline_check_ints(const BatchGeom& g);
// narrow layers (H <= 64, FAST precision): rows on the TMEM lanes, 128-row tiles
bool batchrt_geometry(int64_t N, int D, int H, int n_sms, BatchGeom* g);
size_t batchrt_tile_bytes(const BatchGeom& g);
cudaError_t launch_batchrt_pack(const BatchGeom& g, const float* Xp, void* tiles, cudaStream_t st);
cudaError_t launch_batchrt_epoch(const BatchGeom& g, const void* tiles, const float* Wk, float* part, cudaStream_t st,
                                 int* dbg = nullptr);

// ------------------------------------------------------------ exact eval
cudaError_t launch_eval_ref64(const float* W1, const float* W2, const float* X, const uint8_t* labels, int64_t N,
                              int D, int H, int K, unsigned long long* counts4, double* loss_part, int nparts,
                              cudaStream_t st);
cudaError_t launch_nonfinite(const float* a, int64_t na, const float* b, int64_t nb, int* flag, cudaStream_t st);
int eval_nparts(int64_t N, int H, int K);  // loss partials of launch_eval_ref64
cudaError_t launch_layer_forward(const float* W, const float* X, int64_t N, int m, int n, float* out, cudaStream_t st,
                                 int* counts = nullptr);
cudaError_t launch_layer_backward(const float* x, const float* acts, const double* err, int n, int m, double* deltas,
                                  double* grads, cudaStream_t st, int* counts = nullptr);
cudaError_t launch_forward_pair_debug(const float* W1, const float* W2, const float* x, int D, int H, int K,
                                      float* hidden, float* out, int* stamps, int* status, int workers,
                                      cudaStream_t st);
cudaError_t launch_backprop_error(const float* W, const double* deltas, int n, int m, double* err_prev,
                                  cudaStream_t st);
cudaError_t launch_forward(const float* W1, const float* W2, const float* X, int64_t N, int D, int H, int K,
                           float* hidden, float* out, cudaStream_t st);
cudaError_t launch_instance_gradients(const float* W2, const float* x, const float* hidden, const float* out,
                                      double target, int D, int H, double* g_ih, double* g_ho, cudaStream_t st);
// numpy PCG64 streams on the device (glx_data.cu); st4 = state hi, lo, inc hi, lo
cudaError_t launch_pcg64_f32(const uint64_t* st4, int64_t first, int64_t n_floats, float* out, cudaStream_t st);
cudaError_t launch_pcg64_coin(const uint64_t* st4, int64_t first, int64_t n, uint8_t* labels, cudaStream_t st);
cudaError_t launch_planted_score(const float* X, int64_t N, int D, const int* pick, const double* coef, int k,
                                 double* score, cudaStream_t st);
cudaError_t launch_label_ge(const double* score, int64_t N, const double* thr, uint8_t* labels, cudaStream_t st);
cudaError_t launch_eval_finish(const double* loss_part, int nparts, double* loss_out, cudaStream_t st);

// ------------------------------------------------------------ tcgen05 GEMM
// D[M x N] = A[M x K] . B[N x K]^T, bf16 row-major operands, f32 accumulation in
// TMEM. epi 0: D f32 (ldd); epi 1: bf16 sigmoid(D + bias[col]) into d_bf16 (ldd).
cudaError_t launch_tc_gemm(const void* A, const void* B, int M, int N, int K, int epi, float* d_f32, void* d_bf16,
                           const float* bias, int ldd, cudaStream_t st);

// wide configuration (1024 -> 1024 -> 16) on the tcgen05 GEMM
constexpr int64_t kWideP = 1024 * 1025 + 16 * 1025;  // weights of the wide network
cudaError_t launch_wide_gen(void* Xb, void* XT, uint8_t* labels, int64_t N, uint64_t seed, int64_t row0,
                            cudaStream_t st);
size_t wide_work_bytes(int64_t C, int splits);
int wide_launches_per_chunk();
int wide32_launches_per_chunk();  // the tf32 wide epoch (4 fused, 5 unfused)  // tcgen05 launches per row chunk of the bf16 wide epoch (3 fused, 5 unfused)
cudaError_t wide_grad(const float* W1, const float* W2, const void* Xb, const void* XT, const uint8_t* labels,
                      int64_t N, unsigned char* work, int64_t C, int splits, double* grad, cudaStream_t st,
                      const std::function<void(bool)>& prof);
cudaError_t wide_apply(float* W1, float* W2, const double* grad, double lr_over_n, int* nonfinite, cudaStream_t st);
cudaError_t wide_epoch(float* W1, float* W2, const void* Xb, const void* XT, const uint8_t* labels, int64_t N,
                       double lr, unsigned char* work, int64_t C, int splits, double* stats, int* nonfinite,
                       cudaStream_t st, const std::function<void(bool)>& prof);
// the tf32 variant: f32 rows X [N][1024] and [X,1]^T K-blocked [N/32][1025][32]
cudaError_t launch_wide_gen_tf32(float* X, float* XT, uint8_t* labels, int64_t N, uint64_t seed, int64_t row0,
                                 cudaStream_t st);
size_t wide32_work_bytes(int64_t C, int splits);
cudaError_t wide_grad_tf32(const float* W1, const float* W2, const float* X, const float* XT, const uint8_t* labels,
                           int64_t N, unsigned char* work, int64_t C, int splits, double* grad, cudaStream_t st,
                           const std::function<void(bool)>& prof);
cudaError_t wide_epoch_tf32(float* W1, float* W2, const float* X, const float* XT, const uint8_t* labels, int64_t N,
                            double lr, unsigned char* work, int64_t C, int splits, double* stats, int* nonfinite,
                            cudaStream_t st, const std::function<void(bool)>& prof);

// any-shape engines (glx_generic.cu): online SGD for D > 63 or H > 512, the
// full-batch gradient for shapes outside the batch kernels' register tiles
struct GenNet {
    float* w_ih;  // H x (D+1)
    float* w_ho;  // H + 1
    int H;
    int pad;
};
constexpr size_t kGenMaxSmem = 200 * 1024;
size_t online_generic_smem(int D, int H);
cudaError_t launch_online_generic(const GenNet* nets, int n_nets, int max_h, const float* X, const float* T, int64_t N,
                                  int D, int64_t epochs, double lr, bool ref64, cudaStream_t st);
size_t generic_chunk_rows(int64_t N, int H);
size_t generic_work_bytes(int64_t N, int D, int H);
// grad (f64, glx_batch_grad layout: H(D+1) dW1 sums, H + 1 dW2 sums, loss, tp,
// tn, fp, fn) of the packed rows Xp [N][LD] under (W1, W2)
cudaError_t generic_batch_grad(const float* W1, const float* W2, const float* Xp, int64_t N, int D, int H, int LD,
                               void* work, double* grad, cudaStream_t st);

// ------------------------------------------------------------ diagnostics
cudaError_t launch_fp32_peak(float* out, int iters, int blocks, cudaStream_t st);

}  // namespace glx
