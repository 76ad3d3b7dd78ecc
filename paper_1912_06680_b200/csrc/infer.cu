// infer.cu -- NEXT-3: one forward-pass inference step at the rollout batch ("forward
// passes in larger batches of approximately 60"): LSTM step from the carried state (P:1210,
// P:1202), the heads and masked factorised sampling (reading Q22).
//
//   infer_state   HO[b] = [bf16(h_b) | 1 | 0..] (skipped when HO already holds the state)
//   infer_gates   tcgen05 split-K GEMM: Zp[s][b][r] = W_xh_aug[r, ks] . [x_b | HO_b][ks] -- x
//                 read by TMA straight from the caller's buffer                  (tc_path.cu)
//   infer_cell    z = sum_s Zp[s]; LSTM cell; h, c (fp32 state, in place); HO[b] = bf16(h')
//   infer_heads   tcgen05 split-K GEMM: Yp[s][b][a] = W_o_aug[a, ks] . HO[b, ks]
//   infer_sample  y = sum_s Yp[s]; Gumbel-max per head (primary masked by avail); target-type
//                 table -> head_on; behaviour log-prob of the read heads; value.
// The step streams W (4H x (D+H+64) + A x (H+64) bf16, ~276 MB at the paper's size) once: it
// is HBM-bound on the weights (NEXT-3).
#include "kernels.cuh"

namespace ppo {
namespace {

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

struct InferLayout {
  size_t ho, zp, yp, sched, total;
};
InferLayout infer_layout(const Shape& s, int64_t B) {
  InferLayout L;
  const size_t S = (size_t)tc_infer_max_split();
  L.ho = 0;
  L.zp = align_up(L.ho + (size_t)B * s.Ko * 2, 1024);
  L.yp = align_up(L.zp + S * s.G4 * B * 4, 1024);
  L.sched = align_up(L.yp + S * s.A * B * 4, 1024);
  L.total = align_up(L.sched + kSchedBytes, 1024);
  return L;
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Gumbel(0,1) noise of logit k for row b (reading Q22): u on the 23-bit grid (exact in fp32)
__device__ __forceinline__ float gumbel_noise(uint64_t base, int64_t b, int k) {
  const uint64_t z = splitmix64(base + 1024ull * (uint64_t)b + (uint64_t)k);
  const float u = ((float)(z >> 41) + 0.5f) * 0x1p-23f;
  return -logf(-logf(u));
}

// HO[b] = [bf16(h_b) | 1 | 0...]: the recurrent half of the gates GEMM's batch operand and the
// heads GEMM's.  One thread per 8 columns (16-byte stores), all rows in one flat grid.
__global__ void __launch_bounds__(256) infer_state_kernel(Shape s, int64_t B,
                                                          const float* __restrict__ h,
                                                          __nv_bfloat16* __restrict__ ho) {
  pdl_launch_dependents();
  pdl_wait();
  const int64_t per_row = s.Ko / 8;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B * per_row) return;
  const int64_t b = e / per_row;
  const int64_t col = 8 * (e - b * per_row);
  uint4 v;
  if (col < s.H) {
    const float4* hp = reinterpret_cast<const float4*>(h + b * s.H + col);
    const float4 a = hp[0], c = hp[1];
    __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y), p1 = __floats2bfloat162_rn(a.z, a.w);
    __nv_bfloat162 p2 = __floats2bfloat162_rn(c.x, c.y), p3 = __floats2bfloat162_rn(c.z, c.w);
    v.x = *reinterpret_cast<uint32_t*>(&p0);
    v.y = *reinterpret_cast<uint32_t*>(&p1);
    v.z = *reinterpret_cast<uint32_t*>(&p2);
    v.w = *reinterpret_cast<uint32_t*>(&p3);
  } else {
    v = make_uint4(col == s.H ? 0x3F80u : 0u, 0u, 0u, 0u);   // [1 | 0 ...] (bf16 1.0 = 0x3F80)
  }
  *reinterpret_cast<uint4*>(ho + b * s.Ko + col) = v;
}

// z = sum_s Zp[s][b][r] for the 4 gate rows r of unit j (gate-interleaved rows: r = 256*(j/64)
// + 64*gate + j%64); LSTM cell (oracle O4); h, c updated in place; HO[b][j] = bf16(h').
// Thread per (b, j), j fastest: partial, state and HO accesses are all coalesced.
__global__ void __launch_bounds__(256) infer_cell_kernel(Shape s, int64_t B, int S,
                                                         const float* __restrict__ zp,
                                                         float* __restrict__ h,
                                                         float* __restrict__ c,
                                                         __nv_bfloat16* __restrict__ ho,
                                                         unsigned long long* __restrict__ step_ctr) {
  pdl_launch_dependents();
  pdl_wait();
  // device step counter (graph replays): this step draws with *ctr before the increment; the
  // sample kernel (after this one) reads *ctr - 1
  if (step_ctr && blockIdx.x == 0 && threadIdx.x == 0) *step_ctr += 1ull;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= B * s.H) return;
  const int64_t b = e / s.H;
  const int j = (int)(e - b * s.H);
  const size_t slab = (size_t)s.G4 * B;
  const float* p = zp + b * s.G4 + 256 * (j / 64) + j % 64;
  float z[4] = {0.f, 0.f, 0.f, 0.f};
  int sp = 0;
  for (; sp + 2 <= S; sp += 2) {   // two splits per pass: 8 independent loads in flight
    float a[8];
#pragma unroll
    for (int g = 0; g < 4; ++g) {
      a[g] = p[sp * slab + 64 * g];
      a[4 + g] = p[(sp + 1) * slab + 64 * g];
    }
#pragma unroll
    for (int g = 0; g < 4; ++g) z[g] = z[g] + a[g] + a[4 + g];
  }
  for (; sp < S; ++sp)
#pragma unroll
    for (int g = 0; g < 4; ++g) z[g] += p[sp * slab + 64 * g];
  float gi, gf, gg, go, cn, hn;
  cell_fwd(z[0], z[1], z[2], z[3], c[e], gi, gf, gg, go, cn, hn);
  c[e] = cn;
  h[e] = hn;
  ho[b * s.Ko + j] = __float2bfloat16_rn(hn);
}

// One block per row b: y = sum_s Yp[s][b][.]; warp k samples head k by Gumbel-max over its
// allowed logits (primary: avail) with ties to the smallest index and computes its
// log-softmax at the draw; thread 0 then applies the target-type table.
constexpr int kSampleThreads = 1024;   // one thread per output column in the first phase
__global__ void __launch_bounds__(kSampleThreads) infer_sample_kernel(
    Shape s, int64_t B, int S, const float* __restrict__ yp, const uint8_t* __restrict__ avail,
    const uint8_t* __restrict__ table, uint64_t seed, uint64_t step,
    const unsigned long long* __restrict__ step_ctr, int32_t* __restrict__ act,
    uint8_t* __restrict__ head_on, float* __restrict__ logp, float* __restrict__ value,
    float* __restrict__ out) {
  extern __shared__ float ys[];          // [A] outputs, then [n_logits] Gumbel noise
  __shared__ int sact[PPO_MAX_HEADS];
  __shared__ float slp[PPO_MAX_HEADS];
  __shared__ uint8_t sav[64];   // primary head <= 64 actions (check_dims)
  pdl_launch_dependents();
  pdl_wait();
  const int64_t b = blockIdx.x;
  const int A = (int)s.A;
  const size_t slab = (size_t)A * B;
  const uint64_t base = seed + ((step_ctr ? (uint64_t)(*step_ctr - 1ull) : step) << 32);
  for (int k = threadIdx.x; k < A; k += blockDim.x) {
    const float* p = yp + b * A + k;
    float v[kMaxSplitK];
#pragma unroll
    for (int sp = 0; sp < kMaxSplitK; ++sp) v[sp] = sp < S ? p[sp * slab] : 0.f;
    float acc = 0.f;
#pragma unroll
    for (int sp = 0; sp < kMaxSplitK; ++sp) acc += v[sp];   // split order; +0 beyond S
    ys[k] = acc;
    if (out) out[b * A + k] = acc;
    // the noise of every logit, drawn by the whole block (not by the 7 head warps)
    if (k < s.vcol) ys[A + k] = gumbel_noise(base, b, k);
  }
  for (int k = threadIdx.x; k < s.head_off[1]; k += blockDim.x) sav[k] = avail[b * s.head_off[1] + k];
  __syncthreads();
  const float* gs = ys + A;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int hk = warp; hk < s.n_heads; hk += blockDim.x >> 5) {
    const int off = s.head_off[hk], n = s.head_off[hk + 1] - off;
    float best = -INFINITY, mx = -INFINITY;
    int bi = 0x7fffffff;
    for (int k = lane; k < n; k += 32) {
      if (hk == 0 && !sav[k]) continue;
      const float y = ys[off + k];
      const float sc = y + gs[off + k];
      if (sc > best || (sc == best && k < bi)) {
        best = sc;
        bi = k;
      }
      mx = fmaxf(mx, y);
    }
    for (int o = 16; o; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) {
        best = ob;
        bi = oi;
      }
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    float se = 0.f;
    if (mx != -INFINITY)
      for (int k = lane; k < n; k += 32) {
        if (hk == 0 && !sav[k]) continue;
        se += expf(ys[off + k] - mx);
      }
    for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
    if (lane == 0) {
      const bool none = mx == -INFINITY;  // no available primary action (reading Q23)
      sact[hk] = none ? -1 : bi;
      slp[hk] = none ? 0.f : ys[off + bi] - mx - logf(se);
    }
  }
  __syncthreads();
  if (warp == 0) {   // lane k: head k's table bit, outputs; logp = sum over read heads
    const int a0 = sact[0];
    const int k = lane;
    const bool in = k < s.n_heads;
    const int on = in && a0 >= 0 ? table[a0 * s.n_heads + k] != 0 : 0;
    if (in) {
      act[b * s.n_heads + k] = sact[k];
      if (head_on) head_on[b * s.n_heads + k] = (uint8_t)on;
    }
    float lp = on ? slp[k] : 0.f;
    for (int o = 1; o < 32; o <<= 1) lp += __shfl_xor_sync(0xffffffffu, lp, o);
    if (lane == 0) {
      logp[b] = lp;
      if (value) value[b] = ys[s.vcol];
    }
  }
}

// Inference weight tiling: tile t of a matrix [M][K] (row-major, ld K) = rows 128*(t / nkb)..,
// columns 64*(t % nkb).. as a contiguous [128][64] block (zero beyond M).  One thread per 16 B.
__global__ void __launch_bounds__(256) tile_weights_kernel(const __nv_bfloat16* __restrict__ w,
                                                           int64_t M, int64_t K,
                                                           __nv_bfloat16* __restrict__ wt,
                                                           int64_t n16) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n16;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t nkb = K / 64;
    const int64_t t = e / 1024, r = (e / 8) % 128, c8 = e % 8;
    const int64_t m = (t / nkb) * 128 + r, k = (t % nkb) * 64 + 8 * c8;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (m < M) v = *reinterpret_cast<const uint4*>(w + m * K + k);
    reinterpret_cast<uint4*>(wt)[e] = v;
  }
}

}  // namespace
}  // namespace ppo

using namespace ppo;

extern "C" {

int ppo_infer_ws_bytes(const ppo_dims* dims, int64_t B, size_t* bytes) {
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (B < 1) return fail(PPO_E_SHAPE, "B must be >= 1");
  if (!bytes) return fail(PPO_E_ARG, "bytes is NULL");
  *bytes = infer_layout(s, B).total;
  return PPO_OK;
}

int ppo_infer_weights_bytes(const ppo_dims* dims, size_t* bytes) {
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (!bytes) return fail(PPO_E_ARG, "bytes is NULL");
  *bytes = tc_infer_tiled_elems(s) * 2;
  return PPO_OK;
}

int ppo_infer_pack_weights(const ppo_dims* dims, const void* w, void* wt, size_t wt_bytes,
                           ppo_stream_t st_) {
  cudaStream_t st = (cudaStream_t)st_;
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (!s.bf16) return fail(PPO_E_ARG, "inference weights are bf16 (PPO_PREC_BF16)");
  if (!w || !wt || !aligned(w, 16) || !aligned(wt, 16))
    return fail(PPO_E_ALIGN, "w and wt must be non-NULL and 16-byte aligned");
  if (wt_bytes < tc_infer_tiled_elems(s) * 2)
    return fail(PPO_E_ARG, "wt too small (ppo_infer_weights_bytes)");
  const auto* wb = static_cast<const __nv_bfloat16*>(w);
  auto* wtb = static_cast<__nv_bfloat16*>(wt);
  const size_t off = tc_infer_tiled_offset_heads(s);
  ProfScope _prof("infer_tile_weights", st);
  const int64_t n1 = (int64_t)off / 8, n2 = (int64_t)(tc_infer_tiled_elems(s) - off) / 8;
  tile_weights_kernel<<<(unsigned)std::min<int64_t>((n1 + 255) / 256, 1 << 20), 256, 0, st>>>(
      wb, s.G4, s.Kx, wtb, n1);
  PPO_LAUNCH_CHECK("tile_weights_kernel");
  tile_weights_kernel<<<(unsigned)std::min<int64_t>((n2 + 255) / 256, 1 << 20), 256, 0, st>>>(
      wb + s.G4 * s.Kx, s.A, s.Ko, wtb + off, n2);
  PPO_LAUNCH_CHECK("tile_weights_kernel");
  return PPO_OK;
}

static int infer_impl(const ppo_dims* dims, const void* w, const void* x, float* h, float* c,
                      const uint8_t* avail, const uint8_t* head_table, uint64_t seed,
                      uint64_t step, unsigned long long* step_ctr, uint32_t flags, int64_t B,
                      void* ws, size_t ws_bytes, int32_t* act, uint8_t* head_on, float* logp,
                      float* value, float* out, ppo_stream_t st_) {
  cudaStream_t st = (cudaStream_t)st_;
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (!s.bf16) return fail(PPO_E_ARG, "ppo_infer_step runs the bf16 tensor-core path only");
  if (B < 1 || B > (1 << 22)) return fail(PPO_E_SHAPE, "B must be in [1, 2^22]");
  if (!w || !x || !h || !c || !avail || !head_table || !act || !logp)
    return fail(PPO_E_ARG, "NULL pointer");
  if (!aligned(w, 16) || !aligned(x, 16) || !aligned(h, 16) || !aligned(c, 16))
    return fail(PPO_E_ALIGN, "w, x, h, c must be 16-byte aligned");
  if (!ws || !aligned(ws, 1024)) return fail(PPO_E_ALIGN, "ws must be 1024-byte aligned");
  InferLayout L = infer_layout(s, B);
  if (ws_bytes < L.total) return fail(PPO_E_ARG, "workspace too small (ppo_infer_ws_bytes)");
  if ((rc = check_tc_device())) return rc;
#ifdef PPO_EXPERIMENTS
  // experiment knob (timing breakdowns only; results are wrong when set): skip kernels by bit
  // 1 state, 2 gates GEMM, 4 cell, 8 heads GEMM, 16 sample.  Not in release builds.
  static const int skip = knob_int("PPO_INFER_SKIP", 0);
#else
  constexpr int skip = 0;
#endif
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  auto* ho = reinterpret_cast<__nv_bfloat16*>(wsb + L.ho);
  auto* zp = reinterpret_cast<float*>(wsb + L.zp);
  auto* yp = reinterpret_cast<float*>(wsb + L.yp);
  if (!(flags & PPO_INFER_STATE_CURRENT) && !(skip & 1)) {
    ProfScope _prof("infer_state", st);
    PPO_CUDA_CHECK(launch_pdl(infer_state_kernel, dim3((unsigned)((B * (s.Ko / 8) + 255) / 256)),
                              dim3(256), 0, st, s, B, (const float*)h, ho));
    PPO_LAUNCH_CHECK("infer_state_kernel");
  }
  auto* sched = reinterpret_cast<unsigned int*>(wsb + L.sched);
  if (!(flags & PPO_INFER_STATE_CURRENT)) {
    // first step on this workspace (or state re-derived): zero its tile-scheduler counters;
    // afterwards every GEMM leaves its own pair zero, so steady-state steps need no reset
    ProfScope _prof("sched_reset", st);
    PPO_CUDA_CHECK(cudaMemsetAsync(sched, 0, kSchedBytes, st));
  }
  int S = 1;
  if (!(skip & 2) && (rc = tc_infer_gates(s, B, w, x, ho, zp, &S, sched, st))) return rc;
  if (!(skip & 4)) {
    ProfScope _prof("infer_cell", st);
    PPO_CUDA_CHECK(launch_pdl(infer_cell_kernel, dim3((unsigned)((B * s.H + 255) / 256)), dim3(256),
                              0, st, s, B, S, (const float*)zp, h, c, ho, step_ctr));
    PPO_LAUNCH_CHECK("infer_cell_kernel");
  }
  int S2 = 1;
  if (!(skip & 8) && (rc = tc_infer_heads(s, B, w, ho, yp, &S2, sched, st))) return rc;
  if (!(skip & 16)) {
    ProfScope _prof("infer_sample", st);
    PPO_CUDA_CHECK(launch_pdl(infer_sample_kernel, dim3((unsigned)B), dim3(kSampleThreads),
                              (s.A + s.vcol) * sizeof(float), st, s, B, S2, (const float*)yp, avail,
                              head_table, seed, step, (const unsigned long long*)step_ctr, act,
                              head_on, logp, value, out));
    PPO_LAUNCH_CHECK("infer_sample_kernel");
  }
  return PPO_OK;
}

int ppo_infer_step(const ppo_dims* dims, const void* w, const void* x, float* h, float* c,
                   const uint8_t* avail, const uint8_t* head_table, uint64_t seed, uint64_t step,
                   int64_t B, void* ws, size_t ws_bytes, int32_t* act, uint8_t* head_on,
                   float* logp, float* value, float* out, ppo_stream_t st) {
  return infer_impl(dims, w, x, h, c, avail, head_table, seed, step, nullptr, 0u, B, ws,
                    ws_bytes, act, head_on, logp, value, out, st);
}

int ppo_infer_step_ctr(const ppo_dims* dims, const void* w, const void* x, float* h, float* c,
                       const uint8_t* avail, const uint8_t* head_table, uint64_t seed,
                       uint64_t* step_ctr, uint32_t flags, int64_t B, void* ws,
                       size_t ws_bytes, int32_t* act, uint8_t* head_on, float* logp,
                       float* value, float* out, ppo_stream_t st) {
  if (!step_ctr || !aligned(step_ctr, 8)) return fail(PPO_E_ARG, "step_ctr must be a device u64");
  return infer_impl(dims, w, x, h, c, avail, head_table, seed, 0,
                    reinterpret_cast<unsigned long long*>(step_ctr), flags, B, ws, ws_bytes, act,
                    head_on, logp, value, out, st);
}

}  // extern "C"
