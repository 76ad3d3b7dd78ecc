// common.cuh -- internal helpers shared by the libppo5 translation units.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <utility>

#include "../../include/ppo5.h"

#include <algorithm>

#include <cstdlib>

namespace ppo {

// Fused DP exchange, push mode (comm.cu): where the final gradient of rank `rank` goes --
// element i of theta to stage[i / shard] + rank * shard + i % shard, the owner's slot for
// this rank (CUDA IPC mappings; stage[j] is rank j's staging buffer, world x shard floats).
struct DpStage {
  int world = 0, rank = 0;
  int64_t shard = 0;
  float* stage[PPO_DP_MAX_RANKS] = {};
  __host__ __device__ __forceinline__ float* slot(int64_t i) const {
    const int64_t r = i / shard;
    float* base = stage[0];   // select, not a dynamic index (keeps the param array off the stack)
#pragma unroll
    for (int j = 1; j < PPO_DP_MAX_RANKS; ++j) base = r == j ? stage[j] : base;
    return base + rank * shard + (i - r * shard);
  }
};

// ---- error plumbing (ppo_last_error is thread-local) -----------------------------------
void set_error(const std::string& msg);
int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t e, const char* what);

#define PPO_CUDA_CHECK(expr)                                   \
  do {                                                         \
    cudaError_t _e = (expr);                                   \
    if (_e != cudaSuccess) return ::ppo::cuda_fail(_e, #expr); \
  } while (0)

#define PPO_LAUNCH_CHECK(what)                                  \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::ppo::cuda_fail(_e, what);   \
  } while (0)

// Experiment knobs (A/B timing builds only).  A release build -- the default, what
// build.py produces -- reads no environment variable: knob() is constant NULL and every
// default below is what runs.  Build with -DPPO_EXPERIMENTS (PPO_EXPERIMENTS=1 python
// build.py) to re-enable the PPO_* overrides the tools/ab_variants.py A/B runs use.
#ifdef PPO_EXPERIMENTS
inline const char* knob(const char* name) { return getenv(name); }
#else
inline const char* knob(const char*) { return nullptr; }
#endif
inline int knob_int(const char* name, int def) {
  const char* e = knob(name);
  return e ? atoi(e) : def;
}

inline bool aligned(const void* p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int num_sms();

// ---- tracing: per-launch CUDA events on the launching stream (ppo_prof_start/stop) ---------
void prof_begin(const char* tag, cudaStream_t s);
void prof_end(cudaStream_t s);
struct ProfScope {
  cudaStream_t s;
  ProfScope(const char* tag, cudaStream_t st) : s(st) { prof_begin(tag, st); }
  ~ProfScope() { prof_end(s); }
};

// ---- derived shapes ----------------------------------------------------------------------
struct Shape {
  int64_t D, H, T, A, G4, Kx, Ko;  // G4 = 4H gate rows; A = all head outputs (incl. aux)
  int n_heads;
  int head_off[PPO_MAX_HEADS + 1];
  bool bf16;
  // NEXT-4 aux heads: outputs [vcol + 1, A); A_pass = the output columns whose gradient
  // reaches the LSTM (policy, value, and the win head when win_trunk > 0)
  int vcol, n_win, n_rank, n_bld, n_aux;
  int64_t A_pass;
  float win_trunk;
  bool win_pass;
};
int check_dims(const ppo_dims* d, Shape* s);
int check_tc_device();  // PPO_E_UNSUPPORTED unless an sm_100 device is current

// Launch with programmatic stream serialisation (PDL): the kernel may start while the previous
// kernel on the stream drains; it must execute griddepcontrol.wait before reading its inputs.
template <class... KArgs, class... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Workspace regions (byte offsets from ws base); esz = activation element size.
constexpr int kMaxSplitK = 16;
struct WsLayout {
  size_t xh, g, c, dc, raw, splitk, sched, ready, total;
};
// Dynamic tile-scheduler counters live in the caller's workspace (2 x u32 per GEMM call site),
// so launches on different workspaces -- two optimizers, two streams -- never share one.  The
// call that launches them zeroes them on its stream first; each kernel leaves its pair zero.
enum SchedSlot { kSchedFwd = 0, kSchedHeads, kSchedBwd, kSchedWgrad, kSchedWgradO, kSchedDx,
                 kSchedLstmSlots };
enum InferSchedSlot { kSchedInferGates = 0, kSchedInferHeads, kSchedInferSlots };
constexpr int kSchedWords = 4;       // u32 per slot: die-0 queue, exits, die-1 queue, pad
constexpr size_t kSchedBytes = 128;  // >= kSchedWords * 4 * max(kSchedLstmSlots, kSchedInferSlots)
// SM -> die map of the current device (B200: two dies of ~74 SMs; an L2 line is homed on one
// of them), measured once by a latency probe (tc_path.cu).  NULL if it could not be
// established; *n0 / *n1 = SMs on die 0 / 1.
const uint8_t* sm_die_map(int* n0, int* n1);
WsLayout ws_layout(const Shape& s, int64_t B);
// Multi-step ready counters per (step, 256-row block): one per 64-unit block of the hidden
// state, the row padded to 8 counters (32 bytes, polled as two 16-byte loads).
inline int64_t ready_ld(int64_t H) { return ((std::max<int64_t>(1, (H + 63) / 64) + 7) / 8) * 8; }
inline size_t ready_bytes(int64_t T, int64_t B, int64_t H) {
  return (size_t)T * ((B + 255) / 256) * ready_ld(H) * 4;
}

// ---- activation storage type ---------------------------------------------------------------
__device__ __forceinline__ float to_f(float v) { return v; }
__device__ __forceinline__ float to_f(__nv_bfloat16 v) { return __bfloat162float(v); }
template <class T> __device__ __forceinline__ T from_f(float v);
template <> __device__ __forceinline__ float from_f<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f<__nv_bfloat16>(float v) {
  return __float2bfloat16_rn(v);
}

// ---- the LSTM cell (Gers et al. forget-gate LSTM; oracle O4 / O8) -------------------
__device__ __forceinline__ float sigmoidf_acc(float z) { return 1.0f / (1.0f + expf(-z)); }

// Forward: pre-activations -> gates (i,f,g,o), new cell and hidden state.
__device__ __forceinline__ void cell_fwd(float zi, float zf, float zg, float zo, float c_prev,
                                         float& i, float& f, float& g, float& o, float& c,
                                         float& h) {
  i = sigmoidf_acc(zi);
  f = sigmoidf_acc(zf);
  g = tanhf(zg);
  o = sigmoidf_acc(zo);
  c = f * c_prev + i * g;
  h = o * tanhf(c);
}

// The tensor-core path's cell: the same functions built from the SFU's ex2/rcp (2 MUFU
// instructions each instead of libm's ~25-instruction expf/tanhf and IEEE division), accurate
// to a few 1e-7 -- far below the bf16 storage of the gates and h (2^-9).  tanh takes the odd
// polynomial x - x^3/3 + 2x^5/15 below |x| = 0.1 (error < 6e-9 there), where 1 - e^{-2|x|}
// would cancel.  The fp32 reference path and the inference step keep the libm functions.
__device__ __forceinline__ float ex2_approx(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float sigmoid_tc(float z) {
  return rcp_approx(1.0f + ex2_approx(-1.4426950408889634f * z));
}
__device__ __forceinline__ float tanh_tc(float x) {
  const float a = fabsf(x);
  const float e = ex2_approx(-2.8853900817779268f * a);        // e^{-2|x|}
  const float t = (1.0f - e) * rcp_approx(1.0f + e);
  const float x2 = a * a;
  const float p = a * fmaf(x2, fmaf(x2, 0.13333333333f, -0.33333333333f), 1.0f);
  return copysignf(a < 0.1f ? p : t, x);
}
__device__ __forceinline__ void cell_fwd_tc(float zi, float zf, float zg, float zo, float c_prev,
                                            float& i, float& f, float& g, float& o, float& c,
                                            float& h) {
  i = sigmoid_tc(zi);
  f = sigmoid_tc(zf);
  g = tanh_tc(zg);
  o = sigmoid_tc(zo);
  c = f * c_prev + i * g;
  h = o * tanh_tc(c);
}

// Backward through one cell: dh (total), carried dc, saved gates, c_t, c_{t-1}
// -> pre-activation grads dz (i,f,g,o) and the carry dc_next = dc * f.
__device__ __forceinline__ void cell_bwd(float dh, float dc_carry, float i, float f, float g,
                                         float o, float c, float c_prev, float& dzi, float& dzf,
                                         float& dzg, float& dzo, float& dc_next,
                                         bool tc_math = false) {
  float tc = tc_math ? tanh_tc(c) : tanhf(c);
  float dc = dc_carry + dh * o * (1.0f - tc * tc);
  float d_o = dh * tc;
  float di = dc * g;
  float dg = dc * i;
  float df = dc * c_prev;
  dc_next = dc * f;
  dzi = di * i * (1.0f - i);
  dzf = df * f * (1.0f - f);
  dzg = dg * (1.0f - g * g);
  dzo = d_o * o * (1.0f - o);
}

}  // namespace ppo
