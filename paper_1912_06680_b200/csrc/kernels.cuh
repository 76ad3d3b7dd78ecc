// kernels.cuh -- launcher declarations (internal).
#pragma once
#include "common.cuh"

namespace ppo {

struct LossParams {
  int64_t N;          // rows = T*B
  int A, A_pad, nh;
  int off[PPO_MAX_HEADS + 1];
  float clip_eps, c_v, c_e, inv_denom;
  int vcol, n_win, n_rank, n_aux;        // value column; NEXT-4 aux heads after it
  float c_win, c_rank, c_bld, win_scale; // aux loss weights; win column gradient factor
};

// Operand of the SIMT reference GEMM (see common.cuh Operand); fp32 only.
struct SimtOp {
  const float* p[2];
  int64_t ld[2];
  int64_t rows[2];
  int64_t kext[2];
  int64_t kseg0;
  bool mn;
};

int launch_pack_params(const Shape& s, const float* Wx, const float* Wh, const float* b,
                       const float* Wo, const float* bo, float* theta, int64_t n_wxh,
                       int64_t n_total, cudaStream_t st);
int launch_unpack_params(const Shape& s, const float* theta, float* Wx, float* Wh, float* b,
                         float* Wo, float* bo, int64_t n_wxh, cudaStream_t st);
int launch_cast_bf16(const float* src, void* dst, size_t n, cudaStream_t st);
int launch_pack_x(const Shape& s, int64_t B, const void* x, const float* h0, const float* c0,
                  void* xh, float* c, cudaStream_t st);
constexpr int64_t kGaeShortL = 8192;  // up to this length: one warp per stream
constexpr int64_t kGaeChunk = 4096;   // longer: chunk-parallel look-back kernel
size_t gae_scratch_bytes(int64_t R, int64_t L);
// h0 -> XH[0] h-part, c0 -> C[0], pad columns of every slot (x already in the workspace)
int launch_pack_state(const Shape& s, int64_t B, const float* h0, const float* c0, void* xh,
                      float* c, cudaStream_t st);
// x[i] *= f for i < n (the win-head row fix-up of dW_o, DESIGN Q26)
int launch_scale(float* x, int64_t n, float f, cudaStream_t st);
int launch_gae(const float* rew, const float* val, const uint8_t* done, int64_t R, int64_t L,
               float gamma, float lam, int seq_T, float* adv, float* ret, void* scratch,
               cudaStream_t st);
int launch_loss(const LossParams& p, bool bf16, const float* out, const int32_t* act,
                const uint8_t* head_on, const uint8_t* avail, const float* logp_old,
                const float* adv, const float* ret, const uint8_t* valid, const float* aux_label,
                void* dout, float* logp, float* stats, cudaStream_t st);
struct AdamParams {
  float alpha, b1, omb1, b2, omb2, eps, clip;
  double b1_d, b2_d;   // host copies for the device alpha_t (adam_step_ctr)
};
// a10 on one element (O10): every rounding explicit, so adam_kernel and the
// fused DP kernel (comm.cu) produce the same bits from the same gradient
__device__ __forceinline__ void adam_elem(const AdamParams& ap, float g, float& p, float& m,
                                          float& v) {
  v = __fadd_rn(__fmul_rn(ap.b2, v), __fmul_rn(__fmul_rn(ap.omb2, g), g));
  const float sv = __fsqrt_rn(v);
  const float gc = ap.clip > 0.f ? fminf(fmaxf(g, -__fmul_rn(ap.clip, sv)), __fmul_rn(ap.clip, sv))
                                 : g;
  m = __fadd_rn(__fmul_rn(ap.b1, m), __fmul_rn(ap.omb1, gc));
  p = __fsub_rn(p, __fdiv_rn(__fmul_rn(ap.alpha, m), __fadd_rn(sv, ap.eps)));
}
// host: alpha_t, 1-b1 and 1-b2 formed in double and rounded once to fp32 (ppo5.h adam_step)
inline AdamParams make_adam_params(int64_t t, double lr, double b1, double b2, double eps,
                                   double clip_sigma) {
  AdamParams ap;
  ap.alpha = (float)(lr * sqrt(1.0 - pow(b2, (double)t)) / (1.0 - pow(b1, (double)t)));
  ap.b1 = (float)b1;
  ap.omb1 = (float)(1.0 - b1);
  ap.b2 = (float)b2;
  ap.omb2 = (float)(1.0 - b2);
  ap.eps = (float)eps;
  ap.clip = (clip_sigma > 0.0 && isfinite(clip_sigma)) ? (float)clip_sigma : 0.f;
  ap.b1_d = b1;
  ap.b2_d = b2;
  return ap;
}
// ctr (nullable, device, 16 B): the graph-capturable step counter of adam_step_ctr
int launch_adam(float* p, void* p16, const float* g, float* m, float* v, size_t n,
                const AdamParams& ap, cudaStream_t st, int64_t* ctr = nullptr, double lr = 0.0);
int launch_simt_gemm(const SimtOp& a, const SimtOp& b, int64_t M, int64_t N, int64_t K, float* C,
                     int64_t ldc, cudaStream_t st);
int launch_simt_cell_fwd(const Shape& s, int64_t B, const float* z, const float* c_prev,
                         float* c_out, float* h_out, int64_t ldxh, float* gates, cudaStream_t st);
int launch_simt_cell_bwd(const Shape& s, int64_t B, const float* dh, float* gz, const float* c_t,
                         const float* c_prev, float* dc, cudaStream_t st);

// Cell backward after a split-K dh GEMM: dh = sum of nsplit partials [nsplit][B][H] (fixed
// order), gates -> dz in place in gz [B][4H] (gate-grouped), dc carry in/out (zero if first)
int launch_cell_bwd_split(const float* part, int nsplit, int64_t split_stride, void* gz,
                          const float* c_t, const float* c_prev, float* dc, int64_t B, int64_t H,
                          bool first, cudaStream_t st);
// out[i] = sum_{s < nsplit} part[s * n + i] in fixed order (deterministic split-K reduction)
// dp (nullable): also push the sums to the DP owners' staging (element i = theta dp_base + i)
int launch_splitk_reduce(const float* part, int nsplit, size_t n, float* out, cudaStream_t st,
                         const DpStage* dp = nullptr, int64_t dp_base = 0);

// tcgen05 bf16 path (tc_path.cu)
int tc_forward(const Shape& s, int64_t B, const void* w, void* ws, float* out,
               const cudaEvent_t* x_ready, cudaStream_t st);
// dp (nullable): push the final weight gradients to the DP owners' staging (fused exchange)
// wxh_ready (nullable): recorded on st once the W_xh gradient is final (before dW_o)
int tc_backward(const Shape& s, int64_t B, const void* w, void* ws, const void* dout, float* grad,
                cudaStream_t st, const DpStage* dp = nullptr, cudaEvent_t wxh_ready = nullptr);
// Standalone test GEMM (exported for tests): C = A B^T variants on bf16 inputs.
// NEXT-4: dX = dz W_x over all T*B rows (bf16 path)
int tc_input_grad(const Shape& s, int64_t B, const void* w, void* ws, float* dx, cudaStream_t st);
// NEXT-3: split-K skinny GEMMs of the inference step (weights x batch); *split = partials
int tc_infer_gates(const Shape& s, int64_t B, const void* w, const void* x, const void* ho,
                   float* part, int* split, unsigned int* sched, cudaStream_t st);
int tc_infer_heads(const Shape& s, int64_t B, const void* w, const void* ho, float* part,
                   int* split, unsigned int* sched, cudaStream_t st);
int tc_infer_max_split();
// pre-tiled inference weights: [128][64] bf16 tiles, gates then heads (elements)
size_t tc_infer_tiled_offset_heads(const Shape& s);
size_t tc_infer_tiled_elems(const Shape& s);
int tc_test_gemm(int mode, const void* A, const void* B, float* C, int M, int N, int K,
                 cudaStream_t st);

// ---- vector load/store helpers shared by the HBM-bound kernels
// NV consecutive floats from an arbitrarily aligned p, using aligned 16-byte loads (streaming,
// evict-first); falls back to scalar loads where the aligned window would pass `end`.
template <int NV>
__device__ __forceinline__ void load_floats(const float* p, float (&v)[NV], const float* end) {
  constexpr int NQ = (NV + 6) / 4;
  const int m = static_cast<int>((reinterpret_cast<uintptr_t>(p) >> 2) & 3);
  const float4* b = reinterpret_cast<const float4*>(p - m);
  if (reinterpret_cast<const float*>(b + NQ) <= end) {
    float buf[NQ * 4];
#pragma unroll
    for (int q = 0; q < NQ; ++q) reinterpret_cast<float4*>(buf)[q] = __ldcs(b + q);
    switch (m) {
#define PPO_SHIFT_CASE(M)                                  \
  case M:                                                  \
    _Pragma("unroll") for (int i = 0; i < NV; ++i) v[i] = buf[i + M]; \
    break;
      PPO_SHIFT_CASE(0)
      PPO_SHIFT_CASE(1)
      PPO_SHIFT_CASE(2)
      PPO_SHIFT_CASE(3)
#undef PPO_SHIFT_CASE
    }
  } else {
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = p[i];
  }
}
template <int NV>
__device__ __forceinline__ void store_floats(float* p, const float (&v)[NV]) {
  if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
#pragma unroll
    for (int q = 0; q < NV / 4; ++q)
      reinterpret_cast<float4*>(p)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
#pragma unroll
    for (int i = (NV / 4) * 4; i < NV; ++i) p[i] = v[i];
  } else {
#pragma unroll
    for (int i = 0; i < NV; ++i) p[i] = v[i];
  }
}

}  // namespace ppo
