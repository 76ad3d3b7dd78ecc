// kernels.cu -- HBM-bound kernels of the PPO step (GAE, loss, Adam, layout) and the SIMT
// fp32 reference GEMM path.  See DESIGN.md for the roofline of each.
#include <math.h>
#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"

namespace ppo {

// ============================================================================ layout
// theta layout (ppo5.h): W_xh_aug [4H][Kx] gate-interleaved, W_o_aug [A][Ko].
__device__ __forceinline__ int64_t canon_gate_row(int64_t r, int64_t H) {
  const int64_t q = r >> 8, gate = (r & 255) >> 6, u = r & 63;
  return gate * H + q * 64 + u;
}

__global__ void pack_params_kernel(Shape s, const float* __restrict__ Wx, const float* __restrict__ Wh,
                                   const float* __restrict__ b, const float* __restrict__ Wo,
                                   const float* __restrict__ bo, float* __restrict__ theta,
                                   int64_t n_wxh, int64_t n_total) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n_total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    float v = 0.f;
    if (idx < n_wxh) {
      const int64_t r = idx / s.Kx, c = idx - r * s.Kx;
      const int64_t cr = canon_gate_row(r, s.H);
      if (c < s.D) v = Wx[cr * s.D + c];
      else if (c < s.D + s.H) v = Wh[cr * s.H + (c - s.D)];
      else if (c == s.D + s.H) v = b[cr];
    } else {
      const int64_t i = idx - n_wxh, a = i / s.Ko, c = i - a * s.Ko;
      if (c < s.H) v = Wo[a * s.H + c];
      else if (c == s.H) v = bo[a];
    }
    theta[idx] = v;
  }
}

__global__ void unpack_params_kernel(Shape s, const float* __restrict__ theta, float* __restrict__ Wx,
                                     float* __restrict__ Wh, float* __restrict__ b,
                                     float* __restrict__ Wo, float* __restrict__ bo, int64_t n_wxh) {
  // iterate over theta rows (gate rows of W_xh_aug, then rows of W_o_aug)
  const int64_t nrows = s.G4 + s.A;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       idx < nrows * s.Kx; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = idx / s.Kx, c = idx - r * s.Kx;
    if (r < s.G4) {
      const int64_t cr = canon_gate_row(r, s.H);
      const float v = theta[r * s.Kx + c];
      if (c < s.D) Wx[cr * s.D + c] = v;
      else if (c < s.D + s.H) Wh[cr * s.H + (c - s.D)] = v;
      else if (c == s.D + s.H) b[cr] = v;
    } else {
      const int64_t a = r - s.G4;
      if (c >= s.Ko) continue;
      const float v = theta[n_wxh + a * s.Ko + c];
      if (c < s.H) Wo[a * s.H + c] = v;
      else if (c == s.H) bo[a] = v;
    }
  }
}

__global__ void cast_bf16_kernel(const float* __restrict__ src, __nv_bfloat16* __restrict__ dst,
                                 size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = __float2bfloat16_rn(src[i]);
}

// XH[t][b] = [x_t | h_{t-1} | 1 | 0...] for t = 0..T (x_T := 0), h_{-1} = h0; C[0] = c0.
// One warp per XH row, 16-byte vectors.  The h part of slots t >= 1 is left untouched: the
// forward epilogue of step t-1 writes it.  D, H multiples of 64 keep every segment 16B-aligned.
template <class TA>
__global__ void __launch_bounds__(256) pack_x_kernel(Shape s, int64_t B, const TA* __restrict__ x,
                                                     const float* __restrict__ h0,
                                                     const float* __restrict__ c0,
                                                     TA* __restrict__ xh, float* __restrict__ c) {
  constexpr int V = 16 / sizeof(TA);  // elements per 16-byte vector
  const int lane = threadIdx.x & 31;
  const int64_t rows = (s.T + 1) * B;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows;
       row += nwarps) {
    const int64_t t = row / B, b = row - t * B;
    TA* dst = xh + row * s.Kx;
    uint4* dv = reinterpret_cast<uint4*>(dst);
    if (t < s.T) {
      const uint4* src = reinterpret_cast<const uint4*>(x + (t * B + b) * s.D);
      for (int i = lane; i < s.D / V; i += 32) dv[i] = __ldcs(src + i);
    } else {
      for (int i = lane; i < s.D / V; i += 32) dv[i] = make_uint4(0, 0, 0, 0);
    }
    if (t == 0) {
      const float4* hs = reinterpret_cast<const float4*>(h0 + b * s.H);
      const float4* cs = reinterpret_cast<const float4*>(c0 + b * s.H);
      float4* cd = reinterpret_cast<float4*>(c + b * s.H);
      for (int i = lane; i < s.H / 4; i += 32) {
        const float4 h = hs[i];
        TA* o = dst + s.D + 4 * i;
        o[0] = from_f<TA>(h.x);
        o[1] = from_f<TA>(h.y);
        o[2] = from_f<TA>(h.z);
        o[3] = from_f<TA>(h.w);
        cd[i] = cs[i];
      }
    }
    // [1 | 0 ... 0]: 64 pad columns
    for (int i = lane; i < 64; i += 32) dst[s.D + s.H + i] = from_f<TA>(i == 0 ? 1.f : 0.f);
  }
}

// h0 -> XH[0][b][D:D+H], c0 -> C[0], pad columns [1 | 0...] of all T+1 slots (x is already
// in the workspace).  One warp per XH row.
template <class TA>
__global__ void __launch_bounds__(256) pack_state_kernel(Shape s, int64_t B,
                                                         const float* __restrict__ h0,
                                                         const float* __restrict__ c0,
                                                         TA* __restrict__ xh, float* __restrict__ c) {
  const int lane = threadIdx.x & 31;
  const int64_t rows = (s.T + 1) * B;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows;
       row += nwarps) {
    TA* dst = xh + row * s.Kx;
    if (row < B) {
      const int64_t b = row;
      const float4* hs = reinterpret_cast<const float4*>(h0 + b * s.H);
      const float4* cs = reinterpret_cast<const float4*>(c0 + b * s.H);
      float4* cd = reinterpret_cast<float4*>(c + b * s.H);
      for (int i = lane; i < s.H / 4; i += 32) {
        const float4 h = hs[i];
        TA* o = dst + s.D + 4 * i;
        o[0] = from_f<TA>(h.x);
        o[1] = from_f<TA>(h.y);
        o[2] = from_f<TA>(h.z);
        o[3] = from_f<TA>(h.w);
        cd[i] = cs[i];
      }
    }
    for (int i = lane; i < 64; i += 32) dst[s.D + s.H + i] = from_f<TA>(i == 0 ? 1.f : 0.f);
  }
}

// ============================================================================ GAE

// One warp per rollout stream; windows of 32*CH steps from the end; each lane owns CH steps
// and the affine recurrence A_t = delta_t + c_t A_{t+1} (c_t = gamma lam (1-d_t)) is combined
// across lanes with a reverse shuffle scan of affine maps (oracle O2).  CH = 8 when there are
// enough streams to fill the GPU; CH = 16 doubles the loads in flight per warp otherwise.
// PF = true: the next (earlier) window's loads are issued before this window's scan (more
// registers, more bytes in flight per warp); PF = false: each window loads just before use
// (fewest registers, for launches with enough warps to hide the latency).
template <int CH, bool PF, int MINB = (CH == 8 ? (PF ? 3 : 4) : 1)>
__global__ void __launch_bounds__(256, MINB) gae_kernel(const float* __restrict__ rew, const float* __restrict__ val,
                           const uint8_t* __restrict__ done, int64_t R, int64_t L, float gamma,
                           float lam, int seq_T, float* __restrict__ adv, float* __restrict__ ret,
                           bool vec) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float gl = gamma * lam;
  const int64_t spr = seq_T > 0 ? L / seq_T : 0;  // sequences per rollout
  const int64_t nseq = R * spr;
  for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < R; r += nwarps) {
    const float* rr = rew + r * L;
    const float* vv = val + r * (L + 1);
    const uint8_t* dd = done + r * L;
    float carry = 0.f;
    // Windows of <= W = 32*CH steps from the end.  Lane chunks sit on global multiples of 8
    // steps (window starts are rounded up to them; the row's first window starts its lane 0
    // early and masks the steps before the row), so every full chunk is 32-byte aligned in
    // r, A, R and 8-byte aligned in d, whatever L is.  (V has row stride L + 1: shifted
    // loads.)  Steps outside [w_start, w_end) are identities (delta 0, c 1).
    constexpr int W = 32 * CH;
    const int64_t g0 = r * L;
    const int64_t sh0 = g0 & 7;
    // window [w_start, w_end) and this lane's chunk [t0, t0 + CH) of it
    auto window = [&](int64_t w_end, int64_t& w_start, int64_t& t0, int& i_lo, int& i_hi,
                      bool& full) {
      w_start = w_end - W;
      if (w_start <= 0 && w_end + sh0 <= W) {
        w_start = 0;
      } else {
        if (w_start < 8) w_start = 8;
        w_start += (8 - ((g0 + w_start) & 7)) & 7;
      }
      t0 = w_start - ((g0 + w_start) & 7) + CH * lane;
      i_lo = (int)min((int64_t)CH, max((int64_t)0, w_start - t0));
      i_hi = (int)max((int64_t)0, min((int64_t)CH, w_end - t0));
      full = vec && i_lo == 0 && i_hi == CH;   // vec: bases allow the alignment
    };
    // the next (earlier) window's r, V, d are prefetched while this one computes
    float p_rv[CH], p_v[CH + 1];
    uint2 p_dw[CH / 8];
    auto prefetch = [&](int64_t t0) {
      const float4* r4 = reinterpret_cast<const float4*>(rr + t0);
#pragma unroll
      for (int q = 0; q < CH / 4; ++q) {
        const float4 a4 = __ldcs(r4 + q);
        p_rv[4 * q] = a4.x;
        p_rv[4 * q + 1] = a4.y;
        p_rv[4 * q + 2] = a4.z;
        p_rv[4 * q + 3] = a4.w;
      }
      load_floats<CH + 1>(vv + t0, p_v, val + R * (L + 1));
#pragma unroll
      for (int q = 0; q < CH / 8; ++q) p_dw[q] = __ldcs(reinterpret_cast<const uint2*>(dd + t0) + q);
    };
    int64_t w_end = L, w_start, t0;
    int i_lo, i_hi;
    bool full;
    window(w_end, w_start, t0, i_lo, i_hi, full);
    if (PF && full) prefetch(t0);
    while (w_end > 0) {
      const int n = i_hi;     // (kept for the store path: valid steps are [i_lo, i_hi))
      float delta[CH], cf[CH], vkeep[CH];
      if (full) {
        if (!PF) prefetch(t0);
        float rv[CH], v[CH + 1];
        uint2 dw[CH / 8];
#pragma unroll
        for (int i = 0; i < CH; ++i) rv[i] = p_rv[i];
#pragma unroll
        for (int i = 0; i <= CH; ++i) v[i] = p_v[i];
#pragma unroll
        for (int q = 0; q < CH / 8; ++q) dw[q] = p_dw[q];
        const uint8_t* db = reinterpret_cast<const uint8_t*>(dw);
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          const float nd = db[i] ? 0.f : 1.f;
          delta[i] = rv[i] + gamma * nd * v[i + 1] - v[i];
          cf[i] = gl * nd;
          vkeep[i] = v[i];
        }
      } else {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          if (i >= i_lo && i < i_hi) {
            const int64_t t = t0 + i;
            const float nd = dd[t] ? 0.f : 1.f;
            const float vt = vv[t];
            delta[i] = rr[t] + gamma * nd * vv[t + 1] - vt;
            cf[i] = gl * nd;
            vkeep[i] = vt;
          } else {
            delta[i] = 0.f;
            cf[i] = 1.f;
            vkeep[i] = 0.f;
          }
        }
      }
      // next window: bounds now, its loads in flight during this window's scan and stores
      const int64_t cur_t0 = t0, cur_ws = w_start;
      const int cur_lo = i_lo;
      const bool cur_full = full;
      const int64_t nxt_end = w_start;
      bool nxt_loaded = false;
      if (nxt_end > 0) {
        window(nxt_end, w_start, t0, i_lo, i_hi, full);
        if (PF && full) {
          prefetch(t0);
          nxt_loaded = true;
        }
      }
      float P = 0.f, Q = 1.f;  // A_first = P + Q * A_after
#pragma unroll
      for (int i = CH - 1; i >= 0; --i) {
        P = delta[i] + cf[i] * P;
        Q = cf[i] * Q;
      }
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const float P2 = __shfl_down_sync(0xffffffffu, P, off);
        const float Q2 = __shfl_down_sync(0xffffffffu, Q, off);
        if (lane + off < 32) {
          P = P + Q * P2;
          Q = Q * Q2;
        }
      }
      const float a_first = P + Q * carry;
      float a = __shfl_down_sync(0xffffffffu, a_first, 1);
      if (lane == 31) a = carry;
      float Aout[CH];
#pragma unroll
      for (int i = CH - 1; i >= 0; --i) {
        a = delta[i] + cf[i] * a;
        Aout[i] = a;
      }
      if (seq_T == 0 && cur_full) {
        float Rout[CH];
#pragma unroll
        for (int i = 0; i < CH; ++i) Rout[i] = Aout[i] + vkeep[i];
        store_floats<CH>(adv + r * L + cur_t0, Aout);
        store_floats<CH>(ret + r * L + cur_t0, Rout);
      } else {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          if (i >= cur_lo && i < n) {
            const int64_t t = cur_t0 + i;
            int64_t o;
            if (seq_T > 0) {
              const int64_t k = t / seq_T, tt = t - k * seq_T;
              o = tt * nseq + r * spr + k;
            } else {
              o = r * L + t;
            }
            adv[o] = Aout[i];
            ret[o] = Aout[i] + vkeep[i];   // V_t as loaded (no second read)
          }
        }
      }
      carry = __shfl_sync(0xffffffffu, a_first, 0);
      (void)cur_ws;
      (void)nxt_loaded;
      w_end = nxt_end;
    }
  }
}


// Streams through TMA bulk copies (gae_tma_kernel).  The warp-per-stream kernels above load
// with per-lane vector loads; with few long streams (1,000 x 10^6 steps: ~7 warps per SM) the
// SM's outstanding-miss capacity, not the HBM, caps the bytes in flight (~64 KB per SM).  Here
// lane 0 of each warp streams whole windows (r, V, d of 32*CH steps) into an S-deep
// shared-memory ring with 1-D bulk copies (no per-thread miss tracking), S windows ahead across
// stream boundaries; the lanes then run the same lane-chunk recurrence from shared memory.
// Windows that are not entirely inside the row (the earliest window of a row, when the row is
// not a whole number of windows) or that touch the end of an array take the per-lane load path.
__device__ __forceinline__ void st_global_v8(float* p, const float* v) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0]),
               "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7])
               : "memory");
}
__device__ __forceinline__ uint32_t gae_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
template <int CH, int S, bool FAST>
__global__ void __launch_bounds__(128) gae_tma_kernel(
    const float* __restrict__ rew, const float* __restrict__ val, const uint8_t* __restrict__ done,
    int64_t R, int64_t L, float gamma, float lam, int seq_T, float* __restrict__ adv,
    float* __restrict__ ret, bool vec) {
  constexpr int W = 32 * CH;
  constexpr int RB = W * 4, VB = (W + 8) * 4, DB = W + 16, SB = RB + VB + DB;
  static_assert(SB % 16 == 0, "stage alignment");
  extern __shared__ __align__(128) uint8_t gsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* const wst = gsm + warp * (S * SB + S * 8);
  uint64_t* const bars = reinterpret_cast<uint64_t*>(wst + S * SB);
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(gae_smem(bars + s)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const float gl = gamma * lam;
  const int64_t spr = seq_T > 0 ? L / seq_T : 0, nseq = R * spr;
  // window [w_start, w_end) of row r; wb = its first step on the global 8-step grid
  auto params = [&](int64_t r, int64_t w_end, int64_t& w_start, int64_t& wb, bool& tma) {
    w_start = w_end - W;
    if (w_end < L && w_start >= 8) {
      // a later window's start (already on the 8-step grid) and a whole window before it
      wb = w_start;
      tma = vec && !(r == R - 1 && wb + W + 16 > L);
      return;
    }
    const int64_t g0 = r * L, sh0 = g0 & 7;
    if (w_start <= 0 && w_end + sh0 <= W) {
      w_start = 0;
    } else {
      if (w_start < 8) w_start = 8;
      w_start += (8 - ((g0 + w_start) & 7)) & 7;
    }
    wb = w_start - ((g0 + w_start) & 7);
    // the copies cover [wb, wb + W) (+ slack): steps outside the window belong to the
    // neighbouring rows and are masked by the lanes; only the array's tail is out of bounds
    tma = vec && !(r == R - 1 && wb + W + 16 > L);
  };
  // producer (lane 0): the next window in this warp's order, into stage `st`
  int64_t p_r = gw, p_end = L;
  auto produce = [&](int st) {
    const uint32_t bar = gae_smem(bars + st);
    bool tma = false;
    if (p_r < R) {
      int64_t ws, wb;
      params(p_r, p_end, ws, wb, tma);
      if (tma) {
        uint8_t* s = wst + st * SB;
        const float* rs = rew + p_r * L + wb;
        const float* vs = val + p_r * (L + 1) + wb;
        const uint8_t* ds = done + p_r * L + wb;
        const float* vs_al = reinterpret_cast<const float*>(reinterpret_cast<uintptr_t>(vs) & ~uintptr_t(15));
        const uint8_t* ds_al = reinterpret_cast<const uint8_t*>(reinterpret_cast<uintptr_t>(ds) & ~uintptr_t(15));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(SB)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(gae_smem(s)), "l"(rs), "r"(RB), "r"(bar) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(gae_smem(s + RB)), "l"(vs_al), "r"(VB), "r"(bar) : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(gae_smem(s + RB + VB)), "l"(ds_al), "r"(DB), "r"(bar) : "memory");
      }
      p_end = ws;
      if (p_end == 0) {
        p_r += nwarps;
        p_end = L;
      }
    }
    // windows without a copy (and past the end) still complete the stage's phase
    if (!tma) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
  };
  if (lane == 0) {
#pragma unroll
    for (int s = 0; s < S; ++s) produce(s);
  }
  uint32_t consumed = 0;
  int st = 0;            // stage of window `consumed` (consumed % S) and its phase parity
  uint32_t par = 0;
  for (int64_t r = gw; r < R; r += nwarps) {
    const float* rr = rew + r * L;
    const float* vv = val + r * (L + 1);
    const uint8_t* dd = done + r * L;
    float* const ar = adv + r * L;
    float* const rt = ret + r * L;
    float carry = 0.f;
    int64_t w_end = L;
    while (w_end > 0) {
      int64_t w_start, wb;
      bool tma;
      params(r, w_end, w_start, wb, tma);
      {   // this window's stage phase (a bulk copy, or the producer's plain arrive)
        const uint32_t bar = gae_smem(bars + st);
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "GW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
            "@!p bra GW;\n\t}" ::"r"(bar), "r"(par) : "memory");
      }
      const int64_t t0 = wb + CH * lane;
      // interior window (warp-uniform): every lane's CH steps are in the window and the stage
      // holds them -- no per-step masks, vector stores
      const bool interior = tma && w_start == wb && w_end == wb + W && vec && seq_T == 0;
      float Aout[CH], vkeep[CH], a_first;
      auto window = [&](auto interior_tag) {
        constexpr bool IN = decltype(interior_tag)::value;
        const int i_lo = IN ? 0 : (int)min((int64_t)CH, max((int64_t)0, w_start - t0));
        const int i_hi = IN ? CH : (int)max((int64_t)0, min((int64_t)CH, w_end - t0));
        float delta[CH], cf[CH];
        if (IN || tma) {
          // the lane's chunk out of the stage with 16-byte shared loads (scalar loads at a
          // 4*CH-byte lane stride would be CH-way bank conflicted): r aligned; V shifted by
          // the window's (uniform) misalignment vx; d at byte offset dx in {0, 8}
          const uint8_t* s = wst + st * SB;
          float rv[CH], v[CH + 1];
          const float4* r4 = reinterpret_cast<const float4*>(s) + (CH / 4) * lane;
#pragma unroll
          for (int q = 0; q < CH / 4; ++q) {
            const float4 a4 = r4[q];
            rv[4 * q] = a4.x;
            rv[4 * q + 1] = a4.y;
            rv[4 * q + 2] = a4.z;
            rv[4 * q + 3] = a4.w;
          }
          {
            constexpr int NQ = CH / 4 + 1;   // CH + 1 values starting at vx < 4: NQ float4s
            const int vx = (int)(((reinterpret_cast<uintptr_t>(vv + wb)) & 15) >> 2);
            float buf[NQ * 4];
            const float4* v4 = reinterpret_cast<const float4*>(s + RB) + (CH / 4) * lane;
#pragma unroll
            for (int q = 0; q < NQ; ++q) reinterpret_cast<float4*>(buf)[q] = v4[q];
            switch (vx) {
#define PPO_GAE_VSHIFT(M)                                                     \
  case M:                                                                     \
    _Pragma("unroll") for (int i = 0; i <= CH; ++i) v[i] = buf[i + M]; \
    break;
              PPO_GAE_VSHIFT(0)
              PPO_GAE_VSHIFT(1)
              PPO_GAE_VSHIFT(2)
              PPO_GAE_VSHIFT(3)
#undef PPO_GAE_VSHIFT
            }
          }
          const int dx = (int)((reinterpret_cast<uintptr_t>(dd + wb)) & 15);
          uint8_t db[CH];
          {
            const uint2* d2 = reinterpret_cast<const uint2*>(s + RB + VB + dx) + (CH / 8) * lane;
#pragma unroll
            for (int q = 0; q < CH / 8; ++q) *reinterpret_cast<uint2*>(db + 8 * q) = d2[q];
          }
#pragma unroll
          for (int i = 0; i < CH; ++i) {
            const bool in = IN || (i >= i_lo && i < i_hi);   // window steps (others: identity)
            const float nd = db[i] ? 0.f : 1.f;
            delta[i] = in ? rv[i] + gamma * nd * v[i + 1] - v[i] : 0.f;
            cf[i] = in ? gl * nd : 1.f;
            vkeep[i] = in ? v[i] : 0.f;
          }
        } else {
#pragma unroll
          for (int i = 0; i < CH; ++i) {
            if (i >= i_lo && i < i_hi) {
              const int64_t t = t0 + i;
              const float nd = dd[t] ? 0.f : 1.f;
              const float vt = vv[t];
              delta[i] = rr[t] + gamma * nd * vv[t + 1] - vt;
              cf[i] = gl * nd;
              vkeep[i] = vt;
            } else {
              delta[i] = 0.f;
              cf[i] = 1.f;
              vkeep[i] = 0.f;
            }
          }
        }
        // the stage is read: refill it with the window S ahead (async-proxy write after the
        // generic reads)
        __syncwarp();
        if (lane == 0) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          produce(st);
        }
        float P = 0.f, Q = 1.f;
#pragma unroll
        for (int i = CH - 1; i >= 0; --i) {
          P = delta[i] + cf[i] * P;
          Q = cf[i] * Q;
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const float P2 = __shfl_down_sync(0xffffffffu, P, off);
          const float Q2 = __shfl_down_sync(0xffffffffu, Q, off);
          if (lane + off < 32) {
            P = P + Q * P2;
            Q = Q * Q2;
          }
        }
        a_first = P + Q * carry;
        float a = __shfl_down_sync(0xffffffffu, a_first, 1);
        if (lane == 31) a = carry;
#pragma unroll
        for (int i = CH - 1; i >= 0; --i) {
          a = delta[i] + cf[i] * a;
          Aout[i] = a;
        }
        const bool full = IN || (vec && i_lo == 0 && i_hi == CH);
        if constexpr (IN && CH == 8) {
          // 32-byte aligned (window on the 8-step grid, vec): one 256-bit store per array
          float Rout[CH];
#pragma unroll
          for (int i = 0; i < CH; ++i) Rout[i] = Aout[i] + vkeep[i];
          st_global_v8(ar + t0, Aout);
          st_global_v8(rt + t0, Rout);
        } else if (IN || (seq_T == 0 && full)) {
          float Rout[CH];
#pragma unroll
          for (int i = 0; i < CH; ++i) Rout[i] = Aout[i] + vkeep[i];
          store_floats<CH>(ar + t0, Aout);
          store_floats<CH>(rt + t0, Rout);
        } else {
#pragma unroll
          for (int i = 0; i < CH; ++i) {
            if (i >= i_lo && i < i_hi) {
              const int64_t t = t0 + i;
              int64_t o;
              if (seq_T > 0) {
                const int64_t k = t / seq_T, tt = t - k * seq_T;
                o = tt * nseq + r * spr + k;
              } else {
                o = r * L + t;
              }
              adv[o] = Aout[i];
              ret[o] = Aout[i] + vkeep[i];
            }
          }
        }
      };
      // FAST (long rows): interior windows take the mask-free path; with rows of fewer windows
      // one body measured faster (profiles/r02_gae_fast.txt)
      if constexpr (FAST) {
        if (interior) window(std::true_type{});
        else window(std::false_type{});
      } else {
        window(std::false_type{});
      }
      ++consumed;
      if (++st == S) {
        st = 0;
        par ^= 1u;
      }
      carry = __shfl_sync(0xffffffffu, a_first, 0);
      w_end = w_start;
    }
  }
  // drain: every stage's last phase must complete before the block exits (outstanding copies)
  __syncwarp();
  for (int s = 0; s < S; ++s) {
    const uint32_t c = consumed + (uint32_t)s;
    const uint32_t bar = gae_smem(bars + (c % S));
    const uint32_t par = (c / S) & 1u;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "GD: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra GD;\n\t}" ::"r"(bar), "r"(par) : "memory");
  }
}

// Long rollouts (L > kGaeShortL): chunk-parallel single pass with a decoupled look-back.
// A block owns a chunk of kGaeChunk = 4096 steps of one stream (16 per thread, vectorised).
// Chunks are numbered from the END of each stream and handed out in that order by a global
// counter, so a chunk only waits on chunks dispatched before it.  Each block (1) reduces its
// steps to an affine map A_first = P + Q A_after, (2) publishes it, (3) looks back over the
// later chunks' published maps / inclusive values to get A_after, (4) recomputes its A_t in
// registers, writes A and R, and publishes its inclusive A_first.  r, V, d are read once.
struct GaeStatus {
  float P, Q, A;
  unsigned int flag;  // 0 = empty, 1 = aggregate (P,Q), 2 = inclusive (A)
};

__device__ __forceinline__ void gae_publish(GaeStatus* st, float P, float Q, float A,
                                            unsigned int flag) {
  st->P = P;
  st->Q = Q;
  st->A = A;
  __threadfence();
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&st->flag), "r"(flag) : "memory");
}
__device__ __forceinline__ unsigned int gae_flag(const GaeStatus* st) {
  unsigned int f;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(f) : "l"(&st->flag) : "memory");
  return f;
}

__global__ void __launch_bounds__(256, 3) gae_long_kernel(
    const float* __restrict__ rew, const float* __restrict__ val, const uint8_t* __restrict__ done,
    int64_t R, int64_t L, float gamma, float lam, int seq_T, float* __restrict__ adv,
    float* __restrict__ ret, GaeStatus* __restrict__ status, unsigned int* __restrict__ counter) {
  constexpr int PER = kGaeChunk / 256;
  static_assert(PER % 16 == 0, "done bytes are loaded as 16-byte vectors");
  __shared__ int s_chunk;
  __shared__ float sP[8], sQ[8];
  __shared__ float s_after;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nck = (L + kGaeChunk - 1) / kGaeChunk;  // chunks per stream
  if (tid == 0) s_chunk = (int)atomicAdd(counter, 1u);
  __syncthreads();
  const int64_t g = s_chunk;
  // chunk j (from the end) of every stream before chunk j+1 of any: a chunk's predecessor
  // (chunk j-1 of the same stream, index g - R) was dispatched R blocks earlier
  const int64_t j = g / R, r = g - j * R;
  const int64_t c_end = L - j * kGaeChunk;
  const int64_t c_begin = c_end > kGaeChunk ? c_end - kGaeChunk : 0;
  const int64_t t0 = c_begin + (int64_t)tid * PER;
  const int n = (int)max((int64_t)0, min((int64_t)PER, c_end - t0));
  const float* rr = rew + r * L;
  const float* vv = val + r * (L + 1);
  const uint8_t* dd = done + r * L;
  const float gl = gamma * lam;

  // per step: delta_t, V_t (kept for R_t = A_t + V_t: V is read once) and the done bit (the
  // carry factor gamma lam (1 - d_t) is re-formed from it)
  float delta[PER], vk[PER];
  uint32_t dmask = 0;
  const bool full = n == PER;
  if (full) {
    float rv[PER], v[PER + 1];
    load_floats<PER>(rr + t0, rv, rew + R * L);
    load_floats<PER + 1>(vv + t0, v, val + R * (L + 1));
    uint8_t d[PER];
    if (((reinterpret_cast<uintptr_t>(dd + t0)) & 15) == 0) {
      const uint4* dq = reinterpret_cast<const uint4*>(dd + t0);
#pragma unroll
      for (int q = 0; q < PER / 16; ++q) {
        const uint4 dv = dq[q];
#pragma unroll
        for (int i = 0; i < 16; ++i) d[16 * q + i] = reinterpret_cast<const uint8_t*>(&dv)[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < PER; ++i) d[i] = dd[t0 + i];
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const float nd = d[i] ? 0.f : 1.f;
      delta[i] = rv[i] + gamma * nd * v[i + 1] - v[i];
      vk[i] = v[i];
      dmask |= d[i] ? 1u << i : 0u;
    }
  } else {
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      if (i < n) {
        const int64_t t = t0 + i;
        const float nd = dd[t] ? 0.f : 1.f;
        const float vt = vv[t];
        delta[i] = rr[t] + gamma * nd * vv[t + 1] - vt;
        vk[i] = vt;
        dmask |= dd[t] ? 1u << i : 0u;
      } else {
        delta[i] = 0.f;   // identity step: delta 0, carry factor 1
        vk[i] = 0.f;
      }
    }
  }
  // carry factor of step i: gamma lam (1 - d_i) inside the chunk, 1 past its end
  auto cfac = [&](int i) { return i < n ? ((dmask >> i) & 1u ? 0.f : gl) : 1.f; };
  // (1) thread map, then reverse inclusive scan over the block (later threads are later steps)
  float P = 0.f, Q = 1.f;
#pragma unroll
  for (int i = PER - 1; i >= 0; --i) {
    const float c = cfac(i);
    P = delta[i] + c * P;
    Q = c * Q;
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const float P2 = __shfl_down_sync(0xffffffffu, P, off);
    const float Q2 = __shfl_down_sync(0xffffffffu, Q, off);
    if (lane + off < 32) {
      P = P + Q * P2;
      Q = Q * Q2;
    }
  }
  if (lane == 0) {
    sP[warp] = P;
    sQ[warp] = Q;
  }
  __syncthreads();
  // suffix of the warps after this one
  float wP = 0.f, wQ = 1.f;
  for (int w = 7; w > warp; --w) {
    wP = sP[w] + sQ[w] * wP;
    wQ = sQ[w] * wQ;
  }
  if (tid == 0) {
    // (2) chunk aggregate = warp 0's inclusive map composed with the rest
    const float aP = P + Q * wP, aQ = Q * wQ;
    GaeStatus* me = status + g;
    float after = 0.f;  // A after the last step of the stream (A_L = 0)
    if (j == 0) {
      gae_publish(me, aP, aQ, aP, 2u);
    } else {
      gae_publish(me, aP, aQ, 0.f, 1u);
      // (3) look back over later chunks: compose aggregates until an inclusive value
      float cP = 0.f, cQ = 1.f;  // composed map of the chunks between
      for (int64_t k = g - R;; k -= R) {
        unsigned int f;
        do {
          f = gae_flag(status + k);
        } while (f == 0u);
        const GaeStatus* o = status + k;
        if (f == 2u) {
          after = cP + cQ * *(volatile const float*)&o->A;
          break;
        }
        const float oP = *(volatile const float*)&o->P, oQ = *(volatile const float*)&o->Q;
        cP = cP + cQ * oP;
        cQ = cQ * oQ;
      }
      gae_publish(me, aP, aQ, aP + aQ * after, 2u);
    }
    s_after = after;
  }
  __syncthreads();
  // (4) A after this thread's steps = (warp suffix ∘ lane suffix) applied to the chunk's A_after
  const float a_after_warp = wP + wQ * s_after;
  const float Pn = __shfl_down_sync(0xffffffffu, P, 1), Qn = __shfl_down_sync(0xffffffffu, Q, 1);
  float a = lane == 31 ? a_after_warp : Pn + Qn * a_after_warp;
  float A_out[PER];
#pragma unroll
  for (int i = PER - 1; i >= 0; --i) {
    a = delta[i] + cfac(i) * a;
    A_out[i] = a;
  }
  if (full && seq_T == 0) {
    float vr[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) vr[i] = vk[i] + A_out[i];
    store_floats<PER>(adv + r * L + t0, A_out);
    store_floats<PER>(ret + r * L + t0, vr);
  } else {
    const int64_t spr = seq_T > 0 ? L / seq_T : 0, nseq = R * spr;
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      if (i < n) {
        const int64_t t = t0 + i;
        int64_t o;
        if (seq_T > 0) {
          const int64_t k = t / seq_T, tt = t - k * seq_T;
          o = tt * nseq + r * spr + k;
        } else {
          o = r * L + t;
        }
        adv[o] = A_out[i];
        ret[o] = A_out[i] + vk[i];
      }
    }
  }
}

// ============================================================================ PPO loss
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One warp per row (row = t*B + b); the row is staged in shared memory; per head a masked
// log-sum-exp, the entropy, then the analytic gradient (oracle O6/O7).  Statistics go to
// fixed per-block partial slots and a second kernel reduces them in a fixed order.
template <class TD>
__global__ void __launch_bounds__(256) loss_kernel(
    const float* __restrict__ out, const int32_t* __restrict__ act,
    const uint8_t* __restrict__ head_on, const uint8_t* __restrict__ avail,
    const float* __restrict__ logp_old, const float* __restrict__ adv,
    const float* __restrict__ ret, const uint8_t* __restrict__ valid,
    const float* __restrict__ aux_label, LossParams p, TD* __restrict__ dout,
    float* __restrict__ logp, float* __restrict__ partials) {
  extern __shared__ float smem_y[];
  __shared__ float red[8][PPO_STATS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* y = smem_y + warp * p.A_pad;
  const int A = p.A, nh = p.nh, n0 = p.off[1];
  // stat sums by PPO_STAT_* index; [7] (flags) is kept apart
  float acc[PPO_STATS] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  uint32_t flags = 0;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < p.N; row += (int64_t)gridDim.x * 8) {
    const float* yr = out + row * A;
    if ((A & 3) == 0) {
      const float4* y4 = reinterpret_cast<const float4*>(yr);
      for (int j = lane; j < A / 4; j += 32) reinterpret_cast<float4*>(y)[j] = __ldcs(y4 + j);
    } else {
      for (int j = lane; j < A; j += 32) y[j] = __ldcs(yr + j);
    }
    const uint8_t* av = avail + row * n0;
    const uint32_t m_lo = __ballot_sync(0xffffffffu, lane < n0 && av[lane] != 0);
    const uint32_t m_hi = __ballot_sync(0xffffffffu, lane + 32 < n0 && av[min(lane + 32, n0 - 1)] != 0);
    const uint64_t amask = (uint64_t)m_lo | ((uint64_t)m_hi << 32);
    __syncwarp();
    const float w = valid ? (float)valid[row] : 1.f;
    // per-row metadata loaded lane-parallel once (lane k: head k), broadcast by shuffles
    const int a_l = lane < nh ? act[row * nh + lane] : 0;
    const uint32_t on_l = lane < nh ? head_on[row * nh + lane] : 0u;
    const float lo = logp_old[row], At = adv[row], Rt = ret[row];
    float lse[PPO_MAX_HEADS], Hk[PPO_MAX_HEADS];
    float lpi = 0.f, ent = 0.f;
    for (int k = 0; k < nh; ++k) {
      const int s0 = p.off[k], e0 = p.off[k + 1];
      float mx = -INFINITY;
      for (int j = s0 + lane; j < e0; j += 32)
        if (k != 0 || ((amask >> (j - s0)) & 1ull)) mx = fmaxf(mx, y[j]);
      mx = warp_max(mx);
      // one exp per element: sum e and sum e*y give lse and the entropy
      // H = -sum p log p = lse - sum p y  (p = e / se, log p = y - lse)
      float se = 0.f, sey = 0.f;
      if (mx != -INFINITY)
        for (int j = s0 + lane; j < e0; j += 32)
          if (k != 0 || ((amask >> (j - s0)) & 1ull)) {
            const float e = expf(y[j] - mx);
            se += e;
            sey = fmaf(e, y[j], sey);
          }
      se = warp_sum(se);
      sey = warp_sum(sey);
      const float l = mx == -INFINITY ? 0.f : mx + logf(se);
      const float pl = mx == -INFINITY ? 0.f : sey / se - l;  // sum p log p
      lse[k] = l;
      Hk[k] = -pl;
      const int a = __shfl_sync(0xffffffffu, a_l, k);
      if (__shfl_sync(0xffffffffu, on_l, k)) {
        const int ac = min(max(a, 0), e0 - s0 - 1);
        lpi += y[s0 + ac] - l;
        ent += Hk[k];
      }
      if (k == 0 && w != 0.f) {
        if (amask == 0) flags |= 4u;
        if (a < 0 || a >= n0 || !((amask >> a) & 1ull)) flags |= 2u;
      }
    }
    const float rho = expf(lpi - lo);
    const float s1 = rho * At;
    const float s2 = fminf(fmaxf(rho, 1.f - p.clip_eps), 1.f + p.clip_eps) * At;
    const bool unclipped = s1 <= s2;
    const float pg = -fminf(s1, s2);
    const float V = y[p.vcol];
    const float vf = (V - Rt) * (V - Rt);
    const float lrow = pg + p.c_v * vf - p.c_e * ent;
    const float gpi = unclipped ? -At * rho * w * p.inv_denom : 0.f;
    const float ce = p.c_e * w * p.inv_denom;
    TD* dr = dout + row * A;
    for (int k = 0; k < nh; ++k) {
      const int s0 = p.off[k], e0 = p.off[k + 1];
      const bool on = __shfl_sync(0xffffffffu, on_l, k) != 0u;
      const int a = __shfl_sync(0xffffffffu, a_l, k);
      for (int j = s0 + lane; j < e0; j += 32) {
        float d = 0.f;
        if (on && (k != 0 || ((amask >> (j - s0)) & 1ull))) {
          const float lp = y[j] - lse[k];
          const float pj = expf(lp);
          d = gpi * ((j - s0 == a ? 1.f : 0.f) - pj) + ce * pj * (lp + Hk[k]);
        }
        dr[j] = from_f<TD>(d);
      }
    }
    // NEXT-4 aux heads (oracle aux_loss, DESIGN Q25/Q26): logistic win and building
    // columns lane-parallel, the rank softmax across lanes (n_rank <= 32)
    float laux = 0.f;
    if (p.n_aux) {
      const float* lab = aux_label + row * p.n_aux;
      const int c0 = p.vcol + 1, r0 = p.n_win, r1 = p.n_win + p.n_rank;
      const float wd = w * p.inv_denom;
      for (int j = lane; j < p.n_aux; j += 32) {
        if (j >= r0 && j < r1) continue;
        const float z = y[c0 + j], t = lab[j];
        const float cw = j < r0 ? p.c_win : p.c_bld;
        laux += cw * (fmaxf(z, 0.f) + log1pf(expf(-fabsf(z))) - t * z);
        const float d = cw * wd * (1.f / (1.f + expf(-z)) - t);
        dr[c0 + j] = from_f<TD>(j < r0 ? d * p.win_scale : d);
      }
      if (p.n_rank) {
        const bool in = lane < p.n_rank;
        const float z = in ? y[c0 + r0 + lane] : -INFINITY;
        const float t = in ? lab[r0 + lane] : 0.f;
        const float mx = warp_max(z);
        const float e = in ? expf(z - mx) : 0.f;
        const float se = warp_sum(e);
        const float ty = warp_sum(t);
        const float lse = mx + logf(se);
        if (in) {
          laux += p.c_rank * (-t * (z - lse));
          dr[c0 + r0 + lane] = from_f<TD>(p.c_rank * wd * (e / se * ty - t));
        }
      }
      laux = warp_sum(laux);
    }
    if (lane == 0) {
      dr[p.vcol] = from_f<TD>(2.f * p.c_v * (V - Rt) * w * p.inv_denom);
      if (logp) logp[row] = lpi;
      if (w != 0.f) {
        if (!isfinite(lrow) || !isfinite(laux)) flags |= 1u;
        acc[0] += w * (lrow + laux);
        acc[PPO_STAT_AUX] += w * laux;
        acc[1] += w * pg;
        acc[2] += w * vf;
        acc[3] += w * ent;
        acc[4] += w * (lo - lpi);
        acc[5] += unclipped ? 0.f : w;
        acc[6] += w;
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < PPO_STATS; ++i) red[warp][i] = acc[i];
    red[warp][PPO_STAT_FLAGS] = __uint_as_float(flags);
  }
  __syncthreads();
  if (threadIdx.x < PPO_STATS) {
    const int i = threadIdx.x;
    float v = 0.f;
    uint32_t f = 0;
    for (int wi = 0; wi < 8; ++wi) {
      if (i != PPO_STAT_FLAGS) v += red[wi][i];
      else f |= __float_as_uint(red[wi][i]);
    }
    partials[blockIdx.x * PPO_STATS + i] = i != PPO_STAT_FLAGS ? v : __uint_as_float(f);
  }
}

// ---------------------------------------------------------------------------------------
// The paper's action layout (DESIGN Q17: heads of 30, 4, 189, 189, 81, 81, 81 logits, then the
// value) with compile-time offsets: a warp per row; each lane keeps its 23 logit slots in
// registers for the whole row (one coalesced global read), the 7 per-head reductions run
// interleaved, exp/log are the SFU approximations (ex2/lg2.approx, rel. error ~2^-22), and
// the gradient recomputes p from the registers.  Same arithmetic as loss_kernel (oracle
// O6/O7) with a fraction of its instructions (no per-element index math or branches).
namespace fastloss {
constexpr int NH = 7, NS = 23;
// (closed forms, not recursion: they must fold to constants in the unrolled loops)
__host__ __device__ __forceinline__ constexpr int sz(int k) {   // logits of head k
  return k == 0 ? 30 : k == 1 ? 4 : k <= 3 ? 189 : 81;
}
__host__ __device__ __forceinline__ constexpr int off(int k) {  // first logit of head k
  return k == 0 ? 0 : k == 1 ? 30 : k == 2 ? 34 : k == 3 ? 223 : k == 4 ? 412 : k == 5 ? 493
       : k == 6 ? 574 : 655;
}
__host__ __device__ __forceinline__ constexpr int ni(int k) {   // slots per lane
  return (sz(k) + 31) / 32;
}
__host__ __device__ __forceinline__ constexpr int sb(int k) {   // first slot of head k
  return k == 0 ? 0 : k == 1 ? 1 : k == 2 ? 2 : k == 3 ? 8 : k == 4 ? 14 : k == 5 ? 17
       : k == 6 ? 20 : 23;
}
__host__ __device__ __forceinline__ constexpr int hd(int s) {   // head of slot s
  return s < 1 ? 0 : s < 2 ? 1 : s < 8 ? 2 : s < 14 ? 3 : s < 17 ? 4 : s < 20 ? 5 : 6;
}
__host__ __device__ __forceinline__ constexpr int ix(int s) { return s - sb(hd(s)); }
// slot s of lane l holds logit off(hd(s)) + l + 32 ix(s); it exists iff l < lim(s)
__host__ __device__ __forceinline__ constexpr int lim(int s) { return sz(hd(s)) - 32 * ix(s); }
// packed pairs: slots (s, s+1) of one head with ix(s) even
__host__ __device__ __forceinline__ constexpr bool pair_first(int s) {
  return ix(s) % 2 == 0 && ix(s) + 1 < ni(hd(s));
}
__host__ __device__ __forceinline__ constexpr bool pair_second(int s) { return ix(s) % 2 == 1; }
static_assert(off(1) == sz(0) && off(2) == off(1) + sz(1) && off(3) == off(2) + sz(2) &&
              off(4) == off(3) + sz(3) && off(5) == off(4) + sz(4) &&
              off(6) == off(5) + sz(5) && off(7) == off(6) + sz(6), "offsets");
static_assert(sb(1) == ni(0) && sb(2) == sb(1) + ni(1) && sb(3) == sb(2) + ni(2) &&
              sb(4) == sb(3) + ni(3) && sb(5) == sb(4) + ni(4) && sb(6) == sb(5) + ni(5) &&
              sb(7) == sb(6) + ni(6), "slot bases");
static_assert(sb(NH) == NS && off(NH) == 655, "paper head layout");
constexpr float NEG = -1e30f;   // masked logit (finite: 0 * NEG = 0 in the sums)
constexpr float L2E = 1.4426950408889634f, LN2 = 0.6931471805599453f;
__device__ __forceinline__ float ex2(float x) {
  float r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float lg2(float x) {
  float r;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ float warp_max_redux(float x) {   // sm_100a: one CREDUX
  float r;
  asm("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(x));
  return r;
}
// Sum 16 per-lane values over the warp through a shared-memory transpose: 16 STS, 4 LDS.128,
// 16 FADD and one SHFL (the butterfly reduce-scatter needs 16 SHFL, 30 SEL, 16 FADD).  Lane l
// returns the total of value q = l >> 1 (so value q sits in lanes qlane(q), qlane(q) + 1).
// sc: the warp's [16][36] scratch; row stride 36 keeps each LDS.128 phase conflict-free.
__device__ __forceinline__ float warp_sum16(const float (&v)[16], int lane, float* sc) {
#pragma unroll
  for (int i = 0; i < 16; ++i) sc[i * 36 + lane] = v[i];
  __syncwarp();
  const float4* r = reinterpret_cast<const float4*>(sc + (lane >> 1) * 36 + (lane & 1) * 16);
  const float4 a = r[0], b = r[1], c = r[2], d = r[3];
  __syncwarp();                                 // scratch free for the next row
  const float s = ((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w)) +
                  (((c.x + c.y) + (c.z + c.w)) + ((d.x + d.y) + (d.z + d.w)));
  return s + __shfl_xor_sync(0xffffffffu, s, 1);
}
__host__ __device__ __forceinline__ constexpr int qlane(int q) { return 2 * q; }
}  // namespace fastloss

namespace fastloss {
__device__ __forceinline__ uint32_t su32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// one elected lane: bulk copy (TMA, 1-D) of `bytes` into shared memory, completion counted
// in transaction bytes on the mbarrier at `bar`
__device__ __forceinline__ void bulk_load(uint32_t dst, const void* src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
// one elected lane: bulk copy of `bytes` from shared memory to global (bulk async-group)
__device__ __forceinline__ void bulk_store(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src),
               "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {   // all but the newest N stores have read smem
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra W;\n\t}" ::"r"(bar), "r"(parity) : "memory");
}
constexpr int NBUF = 3;          // row buffers per warp: computing, arriving, draining
constexpr int SCR = 16 * 36;     // per-warp transpose scratch of warp_sum16 (floats)
}  // namespace fastloss

// Each warp walks a contiguous run of rows through three shared-memory row buffers: row r+1
// arrives by TMA bulk copy while row r is computed, and row r-1's dY drains to HBM by a TMA
// bulk store; row r+1's metadata (actions, read flags, availability, logp_old, advantage,
// return) is loaded into registers one row ahead.  Row r's dY is staged in its own buffer (in
// place, once every lane holds its logits in registers).  The grid is one persistent wave
// (SMs x MINB blocks).  Needs A % 4 == 0 and a 16-byte aligned `out` (launch_loss checks).
template <class TD, int MINB>
__global__ void __launch_bounds__(256, MINB) loss_fast_kernel(
    const float* __restrict__ out, const int32_t* __restrict__ act,
    const uint8_t* __restrict__ head_on, const uint8_t* __restrict__ avail,
    const float* __restrict__ logp_old, const float* __restrict__ adv,
    const float* __restrict__ ret, const uint8_t* __restrict__ valid,
    const float* __restrict__ aux_label, LossParams p, TD* __restrict__ dout,
    float* __restrict__ logp, float* __restrict__ partials) {
  using namespace fastloss;
  extern __shared__ __align__(128) float lbuf[];   // [8 warps][NBUF][A], then [8][SCR]
  __shared__ float red[8][PPO_STATS];
  __shared__ __align__(8) uint64_t mbar[8][NBUF];
  constexpr unsigned FULL = 0xffffffffu;
  constexpr int n0 = sz(0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int A = p.A;
  float* const wbuf = lbuf + (size_t)warp * NBUF * A;
  float* const scr = lbuf + (size_t)8 * NBUF * A + warp * SCR;
  const uint32_t rbytes = (uint32_t)A * 4u, obytes = (uint32_t)A * (uint32_t)sizeof(TD);
  const uint32_t buf_s = su32(wbuf), bar_s = su32(&mbar[warp][0]);
  const bool bstore = (obytes & 15) == 0 && (reinterpret_cast<uintptr_t>(dout) & 15) == 0;
  // lane k < 7: head k's first logit and size
  int offl = 0, nl = 1;
#pragma unroll
  for (int k = 0; k < NH; ++k)
    if (lane == k) {
      offl = off(k);
      nl = sz(k);
    }
  float acc[PPO_STATS] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  uint32_t flags = 0;
  const int64_t nw = (int64_t)gridDim.x * 8, gw = (int64_t)blockIdx.x * 8 + warp;
  const int64_t per = (p.N + nw - 1) / nw;
  const int64_t r_beg = min(gw * per, p.N), r_end = min(r_beg + per, p.N);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NBUF; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s + 8 * i) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (r_beg < r_end) bulk_load(buf_s, out + r_beg * A, rbytes, bar_s);
  }
  __syncwarp();
  // metadata, one row ahead: per-lane pointers advance by one row per iteration
  const int32_t* pa = act + r_beg * NH + (lane < NH ? lane : 0);
  const uint8_t* ph = head_on + r_beg * NH + (lane < NH ? lane : 0);
  const uint8_t* pv = avail + r_beg * n0 + (lane < n0 ? lane : 0);
  int a_n = 0;
  uint32_t on_n = 0, av_n = 0;
  float w_n = 1.f, lo_n = 0.f, At_n = 0.f, Rt_n = 0.f;
  auto meta = [&](int64_t r) {
    a_n = lane < NH ? *pa : 0;
    on_n = lane < NH ? *ph : 0u;
    av_n = lane < n0 ? *pv : 0u;
    pa += NH;
    ph += NH;
    pv += n0;
    w_n = valid ? (float)valid[r] : 1.f;
    lo_n = logp_old[r];
    At_n = adv[r];
    Rt_n = ret[r];
  };
  if (r_beg < r_end) meta(r_beg);
  uint32_t phase = 0;                           // bit i: parity of buffer i's next completion
  int b = 0;                                    // buffer of `row`
  for (int64_t row = r_beg; row < r_end; ++row, b = b == NBUF - 1 ? 0 : b + 1) {
    float* const ys = wbuf + b * A;
    const int a_l = a_n;
    const uint32_t on_l = on_n;
    const uint32_t amask = __ballot_sync(FULL, av_n != 0);
    const float w = w_n, lo = lo_n, At = At_n, Rt = Rt_n;
    if (row + 1 < r_end) {
      const int nb = b == NBUF - 1 ? 0 : b + 1;
      if (lane == 0) {
        bulk_wait_read<1>();                    // row - 2's dY store has left buffer nb
        bulk_load(buf_s + nb * rbytes, out + (row + 1) * A, rbytes, bar_s + 8 * nb);
      }
      meta(row + 1);
    }
    const float* yr = out + row * A;
    bar_wait(bar_s + 8 * b, (phase >> b) & 1u);
    phase ^= 1u << b;
    // ---- the row's logits into registers (masked primary entries -> NEG).  After
    // unrolling, hd/ix/off/lim are constants: one base pointer, immediate offsets.
    const float* yl = ys + lane;
    float y[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      bool ok = lim(s) >= 32 || lane < lim(s);
      if (hd(s) == 0) ok = ok && ((amask >> lane) & 1u);
      y[s] = ok ? yl[off(hd(s)) + 32 * ix(s)] : NEG;
    }
    const float ya = lane < NH ? ys[offl + min(max(a_l, 0), nl - 1)] : 0.f;
    const float V = ys[p.vcol];
    __syncwarp();                               // the buffer now becomes row's dY staging
    TD* const ds = reinterpret_cast<TD*>(ys);
    TD* const dl = ds + lane;

    // ---- per-head max (one CREDUX each), then sum e and sum e*y (one SFU exp per element)
    float mx[NH], mb[NH], v[16];
#pragma unroll
    for (int k = 0; k < NH; ++k) mx[k] = NEG;
#pragma unroll
    for (int s = 0; s < NS; ++s) mx[hd(s)] = fmaxf(mx[hd(s)], y[s]);
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      mx[k] = warp_max_redux(mx[k]);
      mb[k] = mx[k] * L2E;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = 0.f;   // v[k] = sum e, v[8 + k] = sum e*y
    // slots of one head in pairs through the packed fp32x2 pipe (FFMA2/FADD2), odd tails alone
    float2 se2[NH], sey2[NH];
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      se2[k] = make_float2(0.f, 0.f);
      sey2[k] = make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int k = hd(s);
      if (pair_first(s)) {
        const float2 y2 = make_float2(y[s], y[s + 1]);
        const float2 a2 = __ffma2_rn(y2, make_float2(L2E, L2E), make_float2(-mb[k], -mb[k]));
        const float2 e2 = make_float2(ex2(a2.x), ex2(a2.y));
        se2[k] = __fadd2_rn(se2[k], e2);
        sey2[k] = __ffma2_rn(e2, y2, sey2[k]);
      } else if (!pair_second(s)) {
        const float e = ex2(fmaf(y[s], L2E, -mb[k]));
        v[k] += e;
        v[8 + k] = fmaf(e, y[s], v[8 + k]);
      }
    }
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      v[k] += se2[k].x + se2[k].y;
      v[8 + k] += sey2[k].x + sey2[k].y;
    }
    // lane l holds the total of value q = l >> 1; the sum-e lanes take sum e*y from lane + 16
    const float tot = warp_sum16(v, lane, scr);
    const float toty = __shfl_xor_sync(FULL, tot, 16);
    const int q = lane >> 1;
    float mq = NEG;
#pragma unroll
    for (int k = 0; k < NH; ++k) mq = q == k ? mx[k] : mq;
    const bool emptyq = mq <= NEG;             // nothing allowed (empty avail)
    const float lse_q = emptyq ? 0.f : mq + lg2(tot) * LN2;
    const float H_q = emptyq ? 0.f : lse_q - toty / tot;
    // ---- log pi(a) and the entropy of the read heads: lane k takes head k; sums over lanes
    // 0..7 (3 butterfly levels), log pi broadcast from lane 0 (the entropy is needed there only)
    const float lsel = __shfl_sync(FULL, lse_q, qlane(lane & 7));
    const float Hl = __shfl_sync(FULL, H_q, qlane(lane & 7));
    float lp_l = 0.f, ent_l = 0.f;
    if (lane < NH && on_l) {
      lp_l = ya - lsel;
      ent_l = Hl;
    }
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      lp_l += __shfl_xor_sync(FULL, lp_l, o);
      ent_l += __shfl_xor_sync(FULL, ent_l, o);
    }
    const float lpi = __shfl_sync(FULL, lp_l, 0), ent = ent_l;
    const int a0 = __shfl_sync(FULL, a_l, 0);
    if (w != 0.f) {
      if (amask == 0) flags |= 4u;
      if (a0 < 0 || a0 >= n0 || !((amask >> a0) & 1u)) flags |= 2u;
    }
    const float rho = __expf(lpi - lo);
    const float s1 = rho * At;
    const float s2 = fminf(fmaxf(rho, 1.f - p.clip_eps), 1.f + p.clip_eps) * At;
    const bool unclipped = s1 <= s2;
    const float pg = -fminf(s1, s2);
    const float vf = (V - Rt) * (V - Rt);
    const float lrow = pg + p.c_v * vf - p.c_e * ent;
    const float gpi = unclipped ? -At * rho * w * p.inv_denom : 0.f;
    const float ce = p.c_e * w * p.inv_denom;
    // ---- dL/dlogits of the read heads: d = p (ce (y - lse + H) - gpi), + gpi at the taken
    // action (stored afterwards by lane k for head k); unread heads and masked entries 0.
    // Lane 2k (holding head k's lse and H) forms head k's coefficients -- exp shift lb, and
    // d = p (cek y + c1) -- and every lane reads all seven back as smem broadcasts.
    const uint32_t on_q = __shfl_sync(FULL, on_l, q & 7);
    float4* const coef = reinterpret_cast<float4*>(scr);
    if (!(lane & 1) && q < NH) {
      const float onf = on_q != 0u ? 1.f : 0.f;
      coef[q] = make_float4(lse_q * L2E, onf * ce, onf * (ce * (H_q - lse_q) - gpi), 0.f);
    }
    __syncwarp();
    float lb[NH], cek[NH], c1[NH];
#pragma unroll
    for (int k = 0; k < NH; ++k) {
      const float4 c = coef[k];
      lb[k] = c.x;
      cek[k] = c.y;
      c1[k] = c.z;
    }
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      const int k = hd(s);
      if (pair_first(s)) {
        const float2 y2 = make_float2(y[s], y[s + 1]);
        const float2 a2 = __ffma2_rn(y2, make_float2(L2E, L2E), make_float2(-lb[k], -lb[k]));
        const float2 t2 = __ffma2_rn(make_float2(cek[k], cek[k]), y2, make_float2(c1[k], c1[k]));
        const float2 d2 = __fmul2_rn(make_float2(ex2(a2.x), ex2(a2.y)), t2);
        if (lim(s) >= 32 || lane < lim(s)) dl[off(k) + 32 * ix(s)] = from_f<TD>(d2.x);
        if (lim(s + 1) >= 32 || lane < lim(s + 1)) dl[off(k) + 32 * ix(s + 1)] = from_f<TD>(d2.y);
      } else if (!pair_second(s)) {
        const float d = ex2(fmaf(y[s], L2E, -lb[k])) * fmaf(cek[k], y[s], c1[k]);
        if (lim(s) >= 32 || lane < lim(s)) dl[off(k) + 32 * ix(s)] = from_f<TD>(d);
      }
    }
    __syncwarp();
    if (lane < NH && on_l) {
      const int a = a_l;
      if (a >= 0 && a < nl && (lane != 0 || ((amask >> a) & 1u))) {
        const float pa = ex2(fmaf(ya, L2E, -lsel * L2E));
        ds[offl + a] = from_f<TD>(pa * fmaf(ce, ya, ce * (Hl - lsel) - gpi) + gpi);
      }
    }
    // ---- NEXT-4 aux heads (as loss_kernel): logistic columns lane-parallel, rank softmax
    float laux = 0.f;
    if (p.n_aux) {
      const float* lab = aux_label + row * p.n_aux;
      const int c0 = p.vcol + 1, r0 = p.n_win, r1 = p.n_win + p.n_rank;
      const float wd = w * p.inv_denom;
      for (int j = lane; j < p.n_aux; j += 32) {
        if (j >= r0 && j < r1) continue;
        const float z = yr[c0 + j], t = lab[j];
        const float cw = j < r0 ? p.c_win : p.c_bld;
        laux += cw * (fmaxf(z, 0.f) + log1pf(expf(-fabsf(z))) - t * z);
        const float dd = cw * wd * (1.f / (1.f + expf(-z)) - t);
        ds[c0 + j] = from_f<TD>(j < r0 ? dd * p.win_scale : dd);
      }
      if (p.n_rank) {
        const bool in = lane < p.n_rank;
        const float z = in ? yr[c0 + r0 + lane] : -INFINITY;
        const float t = in ? lab[r0 + lane] : 0.f;
        const float m = warp_max(z);
        const float e = in ? expf(z - m) : 0.f;
        const float sz_ = warp_sum(e), ty = warp_sum(t);
        const float l = m + logf(sz_);
        if (in) {
          laux += p.c_rank * (-t * (z - l));
          ds[c0 + r0 + lane] = from_f<TD>(p.c_rank * wd * (e / sz_ * ty - t));
        }
      }
      laux = warp_sum(laux);
    }
    if (lane == 0) {
      ds[p.vcol] = from_f<TD>(2.f * p.c_v * (V - Rt) * w * p.inv_denom);
      if (logp) logp[row] = lpi;
      if (w != 0.f) {
        if (!isfinite(lrow) || !isfinite(laux)) flags |= 1u;
        acc[0] += w * (lrow + laux);
        acc[PPO_STAT_AUX] += w * laux;
        acc[1] += w * pg;
        acc[2] += w * vf;
        acc[3] += w * ent;
        acc[4] += w * (lo - lpi);
        acc[5] += unclipped ? 0.f : w;
        acc[6] += w;
      }
    }
    __syncwarp();
    // ---- the staged dY row out: one TMA bulk store (its smem reads are awaited before the
    // buffer is refilled, two rows later)
    TD* const dr = dout + row * A;
    if (bstore) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy
      __syncwarp();
      if (lane == 0) bulk_store(dr, buf_s + b * rbytes, obytes);
    } else {
      __syncwarp();
      for (int i = lane; i < A; i += 32) dr[i] = ds[i];
      // the next bulk load into this buffer is an async-proxy write after these generic reads
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
    }
  }
  if (lane == 0) bulk_wait_read<0>();          // smem stays valid until every store has read it
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < PPO_STATS; ++i) red[warp][i] = acc[i];
    red[warp][PPO_STAT_FLAGS] = __uint_as_float(flags);
  }
  __syncthreads();
  if (threadIdx.x < PPO_STATS) {
    const int i = threadIdx.x;
    float v = 0.f;
    uint32_t f = 0;
    for (int wi = 0; wi < 8; ++wi) {
      if (i != PPO_STAT_FLAGS) v += red[wi][i];
      else f |= __float_as_uint(red[wi][i]);
    }
    partials[blockIdx.x * PPO_STATS + i] = i != PPO_STAT_FLAGS ? v : __uint_as_float(f);
  }
}

// One warp per statistic (9 warps): lane l sums partials l, l+32, ... in order, then a fixed
// xor-shuffle tree -- deterministic, and ~10x shorter than a block-wide loop over the stats.
__global__ void __launch_bounds__(32 * PPO_STATS) loss_finalize_kernel(
    const float* __restrict__ partials, int nblocks, float inv_denom, float* __restrict__ stats) {
  const int i = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float v = 0.f;
  uint32_t f = 0;
  for (int b = lane; b < nblocks; b += 32) {
    const float x = partials[b * PPO_STATS + i];
    if (i != PPO_STAT_FLAGS) v += x;
    else f |= __float_as_uint(x);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    v += __shfl_xor_sync(0xffffffffu, v, o);
    f |= __shfl_xor_sync(0xffffffffu, f, o);
  }
  if (lane == 0) {
    if (i == PPO_STAT_NVALID) stats[i] = v;
    else if (i == PPO_STAT_FLAGS) stats[i] = (float)f;
    else stats[i] = v * inv_denom;
  }
}

// ============================================================================ Adam + clip
// 30 B/param: read p, g, m, v; write p, m, v, bf16 shadow (oracle O10).
// alpha_dev (nullable): alpha_t from the device step counter (adam_tick_kernel), so a
// captured CUDA graph of the step applies the right bias correction on every replay
__global__ void adam_kernel(float* __restrict__ p, __nv_bfloat16* __restrict__ p16,
                            const float* __restrict__ g, float* __restrict__ m,
                            float* __restrict__ v, size_t n, AdamParams ap,
                            const float* __restrict__ alpha_dev) {
  if (alpha_dev) ap.alpha = *alpha_dev;
  const size_t n4 = n / 4;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  // every byte is touched once per step: streaming (evict-first) loads and stores
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += stride) {
    float4 pp = __ldcs(reinterpret_cast<const float4*>(p) + i);
    const float4 gg = __ldcs(reinterpret_cast<const float4*>(g) + i);
    float4 mm = __ldcs(reinterpret_cast<const float4*>(m) + i);
    float4 vv = __ldcs(reinterpret_cast<const float4*>(v) + i);
    float* pe = &pp.x;
    const float* ge = &gg.x;
    float* me = &mm.x;
    float* ve = &vv.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) adam_elem(ap, ge[e], pe[e], me[e], ve[e]);
    __stcs(reinterpret_cast<float4*>(p) + i, pp);
    __stcs(reinterpret_cast<float4*>(m) + i, mm);
    __stcs(reinterpret_cast<float4*>(v) + i, vv);
    if (p16) {
      __nv_bfloat162 lo = __floats2bfloat162_rn(pp.x, pp.y);
      __nv_bfloat162 hi = __floats2bfloat162_rn(pp.z, pp.w);
      uint2 u;
      u.x = *reinterpret_cast<uint32_t*>(&lo);
      u.y = *reinterpret_cast<uint32_t*>(&hi);
      __stcs(reinterpret_cast<uint2*>(p16) + i, u);
    }
  }
  for (size_t i = n4 * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    float pi = p[i], mi = m[i], vi = v[i];
    adam_elem(ap, g[i], pi, mi, vi);
    p[i] = pi;
    m[i] = mi;
    v[i] = vi;
    if (p16) p16[i] = __float2bfloat16_rn(pi);
  }
}

// ============================================================================ SIMT fp32 path
// Reference GEMM C[m][n] = sum_k A(m,k) B(n,k) with FFMA (no tf32), 64x64 tiles.
__device__ __forceinline__ float op_get(const SimtOp& o, int64_t i, int64_t k) {
  int s = k < o.kseg0 ? 0 : 1;
  const int64_t kk = s ? k - o.kseg0 : k;
  if (i >= o.rows[s] || kk >= o.kext[s]) return 0.f;
  const float* p = o.p[s];
  return o.mn ? p[kk * o.ld[s] + i] : p[i * o.ld[s] + kk];
}

__global__ void __launch_bounds__(256) simt_gemm_kernel(SimtOp a, SimtOp b, int64_t M, int64_t N,
                                                        int64_t K, float* __restrict__ C,
                                                        int64_t ldc) {
  __shared__ float As[16][65];
  __shared__ float Bs[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      const int kk = e / 64, ii = e % 64;
      const int64_t k = k0 + kk;
      As[kk][ii] = (k < K && m0 + ii < M) ? op_get(a, m0 + ii, k) : 0.f;
      Bs[kk][ii] = (k < K && n0 + ii < N) ? op_get(b, n0 + ii, k) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        av[i] = As[kk][ty * 4 + i];
        bv[i] = Bs[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) C[m * ldc + n] = acc[i][j];
    }
}

// Cell epilogues for the SIMT path (same cell math as the fused tcgen05 epilogues).
__global__ void simt_cell_fwd_kernel(Shape s, int64_t B, const float* __restrict__ z,
                                     const float* __restrict__ c_prev, float* __restrict__ c_out,
                                     float* __restrict__ h_out, int64_t ldxh,
                                     float* __restrict__ gates) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < B * s.H;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / s.H, j = idx - b * s.H;
    const int64_t base = b * s.G4 + (j >> 6) * 256 + (j & 63);
    float i, f, g, o, c, h;
    cell_fwd(z[base], z[base + 64], z[base + 128], z[base + 192], c_prev[idx], i, f, g, o, c, h);
    c_out[idx] = c;
    h_out[b * ldxh + j] = h;
    gates[base] = i;
    gates[base + 64] = f;
    gates[base + 128] = g;
    gates[base + 192] = o;
  }
}

__global__ void simt_cell_bwd_kernel(Shape s, int64_t B, const float* __restrict__ dh,
                                     float* __restrict__ gz, const float* __restrict__ c_t,
                                     const float* __restrict__ c_prev, float* __restrict__ dc) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < B * s.H;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = idx / s.H, j = idx - b * s.H;
    const int64_t base = b * s.G4 + (j >> 6) * 256 + (j & 63);
    float a, bb, c, d, dn;
    cell_bwd(dh[idx], dc[idx], gz[base], gz[base + 64], gz[base + 128], gz[base + 192], c_t[idx],
             c_prev[idx], a, bb, c, d, dn);
    gz[base] = a;
    gz[base + 64] = bb;
    gz[base + 128] = c;
    gz[base + 192] = d;
    dc[idx] = dn;
  }
}

// ============================================================================ split-K reduce
__global__ void splitk_reduce_kernel(const float4* __restrict__ part, int nsplit, size_t n4,
                                     float4* __restrict__ out, DpStage dp, int64_t dp_base) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4;
       i += (size_t)gridDim.x * blockDim.x) {
    float4 a = part[i];
    for (int sidx = 1; sidx < nsplit; ++sidx) {
      const float4 b = part[sidx * n4 + i];
      a.x += b.x;
      a.y += b.y;
      a.z += b.z;
      a.w += b.w;
    }
    out[i] = a;
    if (dp.world) *reinterpret_cast<float4*>(dp.slot(dp_base + 4 * (int64_t)i)) = a;
  }
}

// ============================================================================ launchers
static int grid_for(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

int launch_pack_params(const Shape& s, const float* Wx, const float* Wh, const float* b,
                       const float* Wo, const float* bo, float* theta, int64_t n_wxh,
                       int64_t n_total, cudaStream_t st) {
  ProfScope _prof("pack_params", st);
  pack_params_kernel<<<grid_for(n_total), 256, 0, st>>>(s, Wx, Wh, b, Wo, bo, theta, n_wxh, n_total);
  PPO_LAUNCH_CHECK("pack_params_kernel");
  return PPO_OK;
}
int launch_unpack_params(const Shape& s, const float* theta, float* Wx, float* Wh, float* b,
                         float* Wo, float* bo, int64_t n_wxh, cudaStream_t st) {
  ProfScope _prof("unpack_params", st);
  unpack_params_kernel<<<grid_for((s.G4 + s.A) * s.Kx), 256, 0, st>>>(s, theta, Wx, Wh, b, Wo, bo, n_wxh);
  PPO_LAUNCH_CHECK("unpack_params_kernel");
  return PPO_OK;
}
int launch_cast_bf16(const float* src, void* dst, size_t n, cudaStream_t st) {
  ProfScope _prof("cast_bf16", st);
  cast_bf16_kernel<<<grid_for((int64_t)n), 256, 0, st>>>(src, (__nv_bfloat16*)dst, n);
  PPO_LAUNCH_CHECK("cast_bf16_kernel");
  return PPO_OK;
}
int launch_pack_x(const Shape& s, int64_t B, const void* x, const float* h0, const float* c0,
                  void* xh, float* c, cudaStream_t st) {
  ProfScope _prof("pack_x", st);
  const int64_t n = (s.T + 1) * B * 32;  // one warp per XH row
  if (s.bf16)
    pack_x_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(
        s, B, (const __nv_bfloat16*)x, h0, c0, (__nv_bfloat16*)xh, c);
  else
    pack_x_kernel<float><<<grid_for(n), 256, 0, st>>>(s, B, (const float*)x, h0, c0, (float*)xh, c);
  PPO_LAUNCH_CHECK("pack_x_kernel");
  return PPO_OK;
}
// Warp-per-stream kernel when streams are short or numerous enough to fill the GPU.
// warp-per-stream kernel unless the streams are too few to fill the GPU with warps
static bool gae_use_short(int64_t R, int64_t L) { return L <= kGaeShortL || R >= 600; }

size_t gae_scratch_bytes(int64_t R, int64_t L) {
  if (gae_use_short(R, L) && knob_int("PPO_GAE_VARIANT", 0) != 5) return 0;
  const int64_t nck = (L + kGaeChunk - 1) / kGaeChunk;
  return 256 + (size_t)(R * nck) * sizeof(GaeStatus);
}
int launch_pack_state(const Shape& s, int64_t B, const float* h0, const float* c0, void* xh,
                      float* c, cudaStream_t st) {
  ProfScope _prof("pack_state", st);
  const int64_t n = (s.T + 1) * B * 32;
  if (s.bf16)
    pack_state_kernel<__nv_bfloat16><<<grid_for(n), 256, 0, st>>>(s, B, h0, c0, (__nv_bfloat16*)xh, c);
  else
    pack_state_kernel<float><<<grid_for(n), 256, 0, st>>>(s, B, h0, c0, (float*)xh, c);
  PPO_LAUNCH_CHECK("pack_state_kernel");
  return PPO_OK;
}
template <int CH, int S, bool FAST>
static int launch_gae_tma_t(const float* rew, const float* val, const uint8_t* done, int64_t R,
                          int64_t L, float gamma, float lam, int seq_T, float* adv, float* ret,
                          bool vec, cudaStream_t st) {
  constexpr int SB = 32 * CH * 4 + (32 * CH + 8) * 4 + 32 * CH + 16;
  constexpr int smem = 4 * (S * SB + S * 8);
  static bool configured = false;
  if (!configured) {
    PPO_CUDA_CHECK(cudaFuncSetAttribute(gae_tma_kernel<CH, S, FAST>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    configured = true;
  }
  const int64_t warps = R;
  static int occ = 0;   // resident blocks per SM at this stage depth (shared memory, registers)
  if (occ == 0) {
    PPO_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, gae_tma_kernel<CH, S, FAST>,
                                                                 128, smem));
    occ = std::max(occ, 1);
  }
  // resident blocks: all that fit for rollouts of a few windows (L = 1,350: 4 blocks per SM
  // 5.54 vs 3 blocks 5.09 TB/s), 3 for longer streams (L = 6,300 / 20,000: 5.70 / 5.55 vs 5.29 /
  // 5.35 TB/s with 4; profiles/r02_gae_persm.txt)
  int per_sm = L <= 2048 ? occ : std::min(occ, 3);
  if (const char* e = knob("PPO_GAE_PER_SM")) per_sm = std::max(1, std::min(occ, atoi(e)));
  // warps per block: 4, or fewer when there are too few streams to give every SM the same
  // number of warps in 4-warp blocks (1,000 streams: 250 blocks = 2 on 102 SMs, 1 on 46)
  int wpb = 4;
  if (warps < (int64_t)num_sms() * per_sm * 4) wpb = knob_int("PPO_GAE_WPB", 4);
  const int blocks = (int)std::min<int64_t>((warps + wpb - 1) / wpb,
                                            (int64_t)num_sms() * per_sm * (4 / wpb));
  gae_tma_kernel<CH, S, FAST><<<blocks, 32 * wpb, smem / 4 * wpb, st>>>(rew, val, done, R, L, gamma,
                                                                  lam, seq_T, adv, ret, vec);
  PPO_LAUNCH_CHECK("gae_tma_kernel");
  return PPO_OK;
}
template <int CH, int S>
static int launch_gae_tma(const float* rew, const float* val, const uint8_t* done, int64_t R,
                          int64_t L, float gamma, float lam, int seq_T, float* adv, float* ret,
                          bool vec, cudaStream_t st) {
  // the second (interior) body pays off only for rows of many windows: L = 10^6 +13%, 10^5
  // +2%, 20,000 even, 6,300 -3.5%, 1,350 -3.5% (profiles/r02_gae_fast.txt)
  if (L >= 65536)
    return launch_gae_tma_t<CH, S, true>(rew, val, done, R, L, gamma, lam, seq_T, adv, ret, vec, st);
  return launch_gae_tma_t<CH, S, false>(rew, val, done, R, L, gamma, lam, seq_T, adv, ret, vec, st);
}
int launch_gae(const float* rew, const float* val, const uint8_t* done, int64_t R, int64_t L,
               float gamma, float lam, int seq_T, float* adv, float* ret, void* scratch,
               cudaStream_t st) {
  ProfScope _prof("gae", st);
  // experiment builds: PPO_GAE_VARIANT = 1 <8, no prefetch>, 2 <8, prefetch>, 3 <16, prefetch>,
  // 4 <16, no prefetch>, 5 the chunk-parallel look-back kernel (needs the long-kernel scratch)
  const int var = knob_int("PPO_GAE_VARIANT", 0);
  if (var >= 1 && var <= 4) {
    const int64_t threads = R * 32;
    const bool vec = aligned(rew, 32) && aligned(done, 8) && aligned(adv, 32) && aligned(ret, 32);
    if (var == 1)
      gae_kernel<8, false><<<grid_for(threads, 256), 256, 0, st>>>(rew, val, done, R, L, gamma, lam,
                                                                   seq_T, adv, ret, vec);
    else if (var == 2)
      gae_kernel<8, true><<<grid_for(threads, 256), 256, 0, st>>>(rew, val, done, R, L, gamma, lam,
                                                                  seq_T, adv, ret, vec);
    else if (var == 3)
      gae_kernel<16, true><<<grid_for(threads, 64), 64, 0, st>>>(rew, val, done, R, L, gamma, lam,
                                                                 seq_T, adv, ret, vec);
    else if (var == 4)
      gae_kernel<16, false><<<grid_for(threads, 256), 256, 0, st>>>(rew, val, done, R, L, gamma,
                                                                    lam, seq_T, adv, ret, vec);
    PPO_LAUNCH_CHECK("gae_kernel");
    return PPO_OK;
  }
  if (var == 6 || var == 7 || var == 8) {   // TMA-streamed windows (CH 16 S 4 / CH 8 S 6 / 8 S 10)
    const bool vec = aligned(rew, 32) && aligned(done, 16) && aligned(val, 16) &&
                     aligned(adv, 32) && aligned(ret, 32);
    if (var == 6) return launch_gae_tma<16, 4>(rew, val, done, R, L, gamma, lam, seq_T, adv, ret,
                                               vec, st);
    if (var == 7) return launch_gae_tma<8, 6>(rew, val, done, R, L, gamma, lam, seq_T, adv, ret,
                                              vec, st);
    return launch_gae_tma<8, 10>(rew, val, done, R, L, gamma, lam, seq_T, adv, ret, vec, st);
  }
  if (var == 0 && gae_use_short(R, L) && L > 256) {
    // several windows per stream: stream them through TMA bulk copies (profiles/
    // r02_gae_variants.txt: +3% at L = 1,350, +5% at 6,300, +15% at 10^5, +7% at 10^6 steps;
    // equal at 20,000); 256-step segments keep the warp kernel below (one window each)
    const bool tvec = aligned(rew, 32) && aligned(done, 16) && aligned(val, 16) &&
                      aligned(adv, 32) && aligned(ret, 32);
    if (tvec) return launch_gae_tma<8, 6>(rew, val, done, R, L, gamma, lam, seq_T, adv, ret, true, st);
  }
  if (var != 5 && gae_use_short(R, L)) {
    const int64_t threads = R * 32;
    // the aligned-chunk path needs 32-byte aligned r, A, R bases and an 8-byte aligned d base
    const bool vec = aligned(rew, 32) && aligned(done, 8) && aligned(adv, 32) && aligned(ret, 32);
    // >= 48 warps per SM (or one window per row): 8-step lane chunks, no prefetch (fewest
    // registers, occupancy hides the latency); 32-48 warps per SM: prefetch the next window
    // during the current one; fewer streams: 16-step chunks with prefetch (four times the
    // loads in flight per warp; 32-step chunks measured slower) in 2-warp blocks spread over
    // all SMs
    if (L <= 256 || R >= 7104)
      gae_kernel<8, false><<<grid_for(threads, 256), 256, 0, st>>>(rew, val, done, R, L, gamma, lam,
                                                               seq_T, adv, ret, vec);
    else if (R >= 4736)
      gae_kernel<8, true><<<grid_for(threads, 256), 256, 0, st>>>(rew, val, done, R, L, gamma,
                                                                  lam, seq_T, adv, ret, vec);
    else
      gae_kernel<16, true><<<grid_for(threads, 64), 64, 0, st>>>(rew, val, done, R, L, gamma,
                                                                 lam, seq_T, adv, ret, vec);
    PPO_LAUNCH_CHECK("gae_kernel");
    return PPO_OK;
  }
  const int64_t nck = (L + kGaeChunk - 1) / kGaeChunk;
  const int64_t blocks = R * nck;
  if (blocks > INT32_MAX) return fail(PPO_E_SHAPE, "too many GAE chunks");
  PPO_CUDA_CHECK(cudaMemsetAsync(scratch, 0, gae_scratch_bytes(R, L), st));
  unsigned int* counter = static_cast<unsigned int*>(scratch);
  GaeStatus* status = reinterpret_cast<GaeStatus*>(static_cast<uint8_t*>(scratch) + 256);
  gae_long_kernel<<<(unsigned)blocks, 256, 0, st>>>(rew, val, done, R, L, gamma, lam, seq_T, adv,
                                                    ret, status, counter);
  PPO_LAUNCH_CHECK("gae_long_kernel");
  return PPO_OK;
}
// one persistent wave (SMs x MINB blocks), two shared-memory row buffers per warp
template <class TD, int MINB>
static int launch_loss_fast(const LossParams& p, const float* out, const int32_t* act,
                            const uint8_t* head_on, const uint8_t* avail, const float* logp_old,
                            const float* adv, const float* ret, const uint8_t* valid,
                            const float* aux_label, void* dout, float* logp, float* partials,
                            int& nblk, cudaStream_t st) {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    PPO_CUDA_CHECK(cudaGetDevice(&dev));
    PPO_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  }
  const size_t smem = 8 * (fastloss::NBUF * (size_t)p.A + fastloss::SCR) * sizeof(float);
  if (smem > 227 * 1024) return fail(PPO_E_SHAPE, "loss: row too wide for the fast kernel");
  if (smem > 48 * 1024)
    PPO_CUDA_CHECK(cudaFuncSetAttribute(loss_fast_kernel<TD, MINB>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  nblk = std::min(PPO_LOSS_BLOCKS, sms * MINB);
  if (const char* g = knob("PPO_LOSS_GRID"))   // experiment knob: grid size
    nblk = std::max(1, std::min(PPO_LOSS_BLOCKS, atoi(g)));
  loss_fast_kernel<TD, MINB><<<nblk, 256, smem, st>>>(out, act, head_on, avail, logp_old, adv,
                                                      ret, valid, aux_label, p, (TD*)dout, logp,
                                                      partials);
  PPO_LAUNCH_CHECK("loss_fast_kernel");
  return PPO_OK;
}
int launch_loss(const LossParams& p, bool bf16, const float* out, const int32_t* act,
                const uint8_t* head_on, const uint8_t* avail, const float* logp_old,
                const float* adv, const float* ret, const uint8_t* valid, const float* aux_label,
                void* dout, float* logp, float* stats, cudaStream_t st) {
  const size_t smem = 8 * (size_t)p.A_pad * sizeof(float);
  float* partials = stats + PPO_STATS;
  int nblk = PPO_LOSS_BLOCKS;
  // the paper's head layout takes the register-resident warp-per-row kernel
  bool fast = p.nh == fastloss::NH && p.vcol == fastloss::off(fastloss::NH);
  for (int k = 0; k <= p.nh && fast; ++k) fast = p.off[k] == fastloss::off(k);
  // rows move by 16-byte TMA bulk copies
  fast = fast && p.A % 4 == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (const char* e = knob("PPO_LOSS_GENERIC")) fast = fast && !atoi(e);
  if (fast) {
    ProfScope _prof("loss", st);
    // 2 blocks of 8 warps per SM: 126 registers and 3 row buffers per warp, no spills
    const int rc = bf16 ? launch_loss_fast<__nv_bfloat16, 2>(p, out, act, head_on, avail,
                                                            logp_old, adv, ret, valid, aux_label,
                                                            dout, logp, partials, nblk, st)
                        : launch_loss_fast<float, 2>(p, out, act, head_on, avail, logp_old, adv,
                                                     ret, valid, aux_label, dout, logp, partials,
                                                     nblk, st);
    if (rc != PPO_OK) return rc;
  } else {
  ProfScope _prof("loss", st);
  if (bf16)
    loss_kernel<__nv_bfloat16><<<PPO_LOSS_BLOCKS, 256, smem, st>>>(
        out, act, head_on, avail, logp_old, adv, ret, valid, aux_label, p, (__nv_bfloat16*)dout,
        logp, partials);
  else
    loss_kernel<float><<<PPO_LOSS_BLOCKS, 256, smem, st>>>(
        out, act, head_on, avail, logp_old, adv, ret, valid, aux_label, p, (float*)dout, logp,
        partials);
  PPO_LAUNCH_CHECK("loss_kernel");
  }
  ProfScope _prof("loss_finalize", st);
  loss_finalize_kernel<<<1, 32 * PPO_STATS, 0, st>>>(partials, nblk, p.inv_denom, stats);
  PPO_LAUNCH_CHECK("loss_finalize_kernel");
  return PPO_OK;
}
__global__ void scale_kernel(float* __restrict__ x, int64_t n, float f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    x[i] *= f;
}
int launch_scale(float* x, int64_t n, float f, cudaStream_t st) {
  ProfScope _prof("scale", st);
  scale_kernel<<<grid_for(n), 256, 0, st>>>(x, n, f);
  PPO_LAUNCH_CHECK("scale_kernel");
  return PPO_OK;
}
// the device step counter of adam_step_ctr: t = ++ctr[0]; alpha_t (O10) formed in double
// and rounded once to fp32, like the host path (ppo5.h adam_step), into the float at ctr + 8 B
__global__ void adam_tick_kernel(long long* ctr, double lr, double b1, double b2) {
  const long long t = ctr[0] + 1;
  ctr[0] = t;
  *reinterpret_cast<float*>(ctr + 1) =
      (float)(lr * sqrt(1.0 - pow(b2, (double)t)) / (1.0 - pow(b1, (double)t)));
}
int launch_adam(float* p, void* p16, const float* g, float* m, float* v, size_t n,
                const AdamParams& ap, cudaStream_t st, int64_t* ctr, double lr) {
  if (ctr) {
    ProfScope _prof("adam_tick", st);
    adam_tick_kernel<<<1, 1, 0, st>>>(reinterpret_cast<long long*>(ctr), lr, (double)ap.b1_d,
                                      (double)ap.b2_d);
    PPO_LAUNCH_CHECK("adam_tick_kernel");
  }
  ProfScope _prof("adam", st);
  adam_kernel<<<grid_for((int64_t)(n / 4 + 1)), 256, 0, st>>>(
      p, (__nv_bfloat16*)p16, g, m, v, n, ap,
      ctr ? reinterpret_cast<const float*>(ctr + 1) : nullptr);
  PPO_LAUNCH_CHECK("adam_kernel");
  return PPO_OK;
}
int launch_splitk_reduce(const float* part, int nsplit, size_t n, float* out, cudaStream_t st,
                         const DpStage* dp, int64_t dp_base) {
  ProfScope _prof("splitk_reduce", st);
  splitk_reduce_kernel<<<grid_for((int64_t)(n / 4)), 256, 0, st>>>(
      reinterpret_cast<const float4*>(part), nsplit, n / 4, reinterpret_cast<float4*>(out),
      dp ? *dp : DpStage{}, dp_base);
  PPO_LAUNCH_CHECK("splitk_reduce_kernel");
  return PPO_OK;
}
int launch_simt_gemm(const SimtOp& a, const SimtOp& b, int64_t M, int64_t N, int64_t K, float* C,
                     int64_t ldc, cudaStream_t st) {
  ProfScope _prof("simt_gemm", st);
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64));
  simt_gemm_kernel<<<grid, 256, 0, st>>>(a, b, M, N, K, C, ldc);
  PPO_LAUNCH_CHECK("simt_gemm_kernel");
  return PPO_OK;
}
int launch_simt_cell_fwd(const Shape& s, int64_t B, const float* z, const float* c_prev,
                         float* c_out, float* h_out, int64_t ldxh, float* gates, cudaStream_t st) {
  ProfScope _prof("simt_cell_fwd", st);
  simt_cell_fwd_kernel<<<grid_for(B * s.H), 256, 0, st>>>(s, B, z, c_prev, c_out, h_out, ldxh, gates);
  PPO_LAUNCH_CHECK("simt_cell_fwd_kernel");
  return PPO_OK;
}
// Cell backward of one recurrent step after a split-K dh GEMM (small minibatches, where the
// step GEMM has fewer tiles than CTA pairs): dh = sum of nsplit fp32 partials (fixed order),
// then the same cell math as the fused EpiLstmBwd epilogue (tc_math sigmoid/tanh), dz over the
// bf16 gates in place and the dc carry.  A thread per (row, 8 units); the 8 threads of a
// 64-unit block read each gate's 128 contiguous bytes (coalesced, unlike the epilogue's
// row-per-thread access).
__global__ void __launch_bounds__(256) cell_bwd_split_kernel(
    const float* __restrict__ part, int nsplit, int64_t split_stride, __nv_bfloat16* gz,
    const float* __restrict__ c_t, const float* __restrict__ c_prev, float* dc, int64_t B,
    int64_t H, int first) {
  const int64_t nch = H / 8;
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= B * nch) return;
  const int64_t m = idx / nch;
  const int64_t j0 = (idx - m * nch) * 8;
  const int64_t o = m * H + j0;
  float dh[8], ct[8], cp[8], dcv[8];
  {
    const float4* p4 = reinterpret_cast<const float4*>(part + o);
    float4 a = p4[0], b = p4[1];
    for (int sp = 1; sp < nsplit; ++sp) {
      const float4* q4 = reinterpret_cast<const float4*>(part + sp * split_stride + o);
      const float4 x = q4[0], y = q4[1];
      a.x += x.x; a.y += x.y; a.z += x.z; a.w += x.w;
      b.x += y.x; b.y += y.y; b.z += y.z; b.w += y.w;
    }
    dh[0] = a.x; dh[1] = a.y; dh[2] = a.z; dh[3] = a.w;
    dh[4] = b.x; dh[5] = b.y; dh[6] = b.z; dh[7] = b.w;
  }
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    const float4 x = reinterpret_cast<const float4*>(c_t + o)[q];
    const float4 y = reinterpret_cast<const float4*>(c_prev + o)[q];
    ct[4 * q] = x.x; ct[4 * q + 1] = x.y; ct[4 * q + 2] = x.z; ct[4 * q + 3] = x.w;
    cp[4 * q] = y.x; cp[4 * q + 1] = y.y; cp[4 * q + 2] = y.z; cp[4 * q + 3] = y.w;
    if (first) {
#pragma unroll
      for (int i = 0; i < 4; ++i) dcv[4 * q + i] = 0.f;
    } else {
      const float4 z = reinterpret_cast<const float4*>(dc + o)[q];
      dcv[4 * q] = z.x; dcv[4 * q + 1] = z.y; dcv[4 * q + 2] = z.z; dcv[4 * q + 3] = z.w;
    }
  }
  // gates of units j0..j0+7: gate q at (j0 >> 6) * 256 + q * 64 + (j0 & 63) (gate-grouped rows)
  __nv_bfloat16* g = gz + m * 4 * H + (j0 >> 6) * 256 + (j0 & 63);
  uint4 graw[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) graw[q] = *reinterpret_cast<const uint4*>(g + q * 64);
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    float z[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const uint32_t u = reinterpret_cast<const uint32_t*>(&graw[q])[w];
      z[q][0] = __uint_as_float(u << 16);
      z[q][1] = __uint_as_float(u & 0xFFFF0000u);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int e = 2 * w + h;
      float a, b, c, d, dn;
      cell_bwd(dh[e], dcv[e], z[0][h], z[1][h], z[2][h], z[3][h], ct[e], cp[e], a, b, c, d, dn,
               true);
      z[0][h] = a;
      z[1][h] = b;
      z[2][h] = c;
      z[3][h] = d;
      dcv[e] = dn;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const __nv_bfloat162 pk = __floats2bfloat162_rn(z[q][0], z[q][1]);
      reinterpret_cast<uint32_t*>(&graw[q])[w] = *reinterpret_cast<const uint32_t*>(&pk);
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(g + q * 64) = graw[q];
#pragma unroll
  for (int q = 0; q < 2; ++q)
    reinterpret_cast<float4*>(dc + o)[q] =
        make_float4(dcv[4 * q], dcv[4 * q + 1], dcv[4 * q + 2], dcv[4 * q + 3]);
}
int launch_cell_bwd_split(const float* part, int nsplit, int64_t split_stride, void* gz,
                          const float* c_t, const float* c_prev, float* dc, int64_t B, int64_t H,
                          bool first, cudaStream_t st) {
  if (H % 64 != 0) return fail(PPO_E_SHAPE, "split cell backward needs H % 64 == 0");
  ProfScope _prof("cell_bwd", st);
  const int64_t threads = B * (H / 8);
  cell_bwd_split_kernel<<<grid_for(threads, 256), 256, 0, st>>>(
      part, nsplit, split_stride, static_cast<__nv_bfloat16*>(gz), c_t, c_prev, dc, B, H,
      first ? 1 : 0);
  PPO_LAUNCH_CHECK("cell_bwd_split_kernel");
  return PPO_OK;
}

int launch_simt_cell_bwd(const Shape& s, int64_t B, const float* dh, float* gz, const float* c_t,
                         const float* c_prev, float* dc, cudaStream_t st) {
  ProfScope _prof("simt_cell_bwd", st);
  simt_cell_bwd_kernel<<<grid_for(B * s.H), 256, 0, st>>>(s, B, dh, gz, c_t, c_prev, dc);
  PPO_LAUNCH_CHECK("simt_cell_bwd_kernel");
  return PPO_OK;
}

}  // namespace ppo
