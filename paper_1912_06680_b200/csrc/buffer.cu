// buffer.cu -- NEXT-1: the optimizer's device-resident experience buffer,
// uniform minibatch sampling and the gather of a minibatch straight into the forward
// workspace (zero-copy inputs for lstm_bptt_fwd).  See include/ppo5.h.
#include "kernels.cuh"

namespace ppo {
namespace {

// splitmix64 (Steele, Lea, Flood 2014): the counter-based generator both this library and the
// oracle implement for minibatch sampling.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void sample_indices_kernel(int64_t capacity, int64_t B, uint64_t seed, uint64_t step,
                                      int32_t* __restrict__ idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < B;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = seed + (step << 32) + static_cast<uint64_t>(i);
    idx[i] = static_cast<int32_t>(splitmix64(key) % static_cast<uint64_t>(capacity));
  }
}

// XH[t][b] = [x(idx[b], t) | h (t=0: h0(idx[b])) | 1 | 0...] for t = 0..T; C[0][b] = c0(idx[b]).
// One warp per XH row, 16-byte vectors.
template <class TA>
__global__ void __launch_bounds__(256) gather_x_kernel(Shape s, int64_t B, const TA* __restrict__ bx,
                                                       const float* __restrict__ bh0,
                                                       const float* __restrict__ bc0,
                                                       const int32_t* __restrict__ idx,
                                                       TA* __restrict__ xh, float* __restrict__ c) {
  constexpr int V = 16 / sizeof(TA);
  const int lane = threadIdx.x & 31;
  const int64_t rows = (s.T + 1) * B;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows;
       row += nwarps) {
    const int64_t t = row / B, b = row - t * B;
    const int64_t src = idx[b];
    TA* dst = xh + row * s.Kx;
    uint4* dv = reinterpret_cast<uint4*>(dst);
    if (t < s.T) {
      const uint4* sv = reinterpret_cast<const uint4*>(bx + (src * s.T + t) * s.D);
      for (int i = lane; i < s.D / V; i += 32) dv[i] = sv[i];
    } else {
      for (int i = lane; i < s.D / V; i += 32) dv[i] = make_uint4(0, 0, 0, 0);
    }
    if (t == 0) {
      const float4* hs = reinterpret_cast<const float4*>(bh0 + src * s.H);
      const float4* cs = reinterpret_cast<const float4*>(bc0 + src * s.H);
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

// Per-timestep loss inputs: buffer [cap][T][.] -> minibatch [T][B][.].
__global__ void gather_rows_kernel(Shape s, int64_t B, const ppo_buffer buf,
                                   const int32_t* __restrict__ idx, int32_t* __restrict__ act,
                                   uint8_t* __restrict__ head_on, uint8_t* __restrict__ avail,
                                   float* __restrict__ logp_old, float* __restrict__ adv,
                                   float* __restrict__ ret, uint8_t* __restrict__ valid) {
  const int nh = s.n_heads, n0 = s.head_off[1];
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < s.T * B;
       r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = r / B, b = r - t * B;
    const int64_t q = static_cast<int64_t>(idx[b]) * s.T + t;  // buffer row
    for (int k = 0; k < nh; ++k) {
      act[r * nh + k] = buf.act[q * nh + k];
      head_on[r * nh + k] = buf.head_on[q * nh + k];
    }
    for (int k = 0; k < n0; ++k) avail[r * n0 + k] = buf.avail[q * n0 + k];
    logp_old[r] = buf.logp_old[q];
    adv[r] = buf.adv[q];
    ret[r] = buf.ret[q];
    if (valid) valid[r] = buf.valid ? buf.valid[q] : 1;
  }
}

int grid_of(int64_t n, int threads = 256) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = (int64_t)num_sms() * 16;
  return (int)std::max<int64_t>(1, std::min(g, cap));
}

}  // namespace
}  // namespace ppo

using namespace ppo;

extern "C" {

int ppo_sample_indices(int64_t capacity, int64_t B, uint64_t seed, uint64_t step, int32_t* idx,
                       ppo_stream_t st) {
  if (capacity < 1 || capacity > INT32_MAX || B < 0) return fail(PPO_E_ARG, "bad capacity/B");
  if (B == 0) return PPO_OK;
  if (!idx) return fail(PPO_E_ARG, "idx is NULL");
  ProfScope _prof("sample_indices", (cudaStream_t)st);
  sample_indices_kernel<<<grid_of(B), 256, 0, (cudaStream_t)st>>>(capacity, B, seed, step, idx);
  PPO_LAUNCH_CHECK("sample_indices_kernel");
  return PPO_OK;
}

int ppo_gather(const ppo_dims* dims, const ppo_buffer* buf, const int32_t* idx, int64_t B,
               void* ws, size_t ws_bytes, int32_t* act, uint8_t* head_on, uint8_t* avail,
               float* logp_old, float* adv, float* ret, uint8_t* valid, ppo_stream_t st_) {
  cudaStream_t st = (cudaStream_t)st_;
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (!buf || !buf->x || !buf->h0 || !buf->c0 || !buf->act || !buf->head_on || !buf->avail ||
      !buf->logp_old || !buf->adv || !buf->ret)
    return fail(PPO_E_ARG, "buffer has NULL arrays");
  if (B < 1) return fail(PPO_E_SHAPE, "B must be >= 1");
  if (!idx || !act || !head_on || !avail || !logp_old || !adv || !ret)
    return fail(PPO_E_ARG, "NULL pointer");
  if (!aligned(buf->x, 16) || !aligned(buf->h0, 16) || !aligned(buf->c0, 16))
    return fail(PPO_E_ALIGN, "buffer x/h0/c0 must be 16-byte aligned");
  if (!ws || !aligned(ws, 1024)) return fail(PPO_E_ALIGN, "ws must be 1024-byte aligned");
  WsLayout L = ws_layout(s, B);
  if (ws_bytes < L.total) return fail(PPO_E_ARG, "workspace too small");
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  float* C = reinterpret_cast<float*>(wsb + L.c);
  {
    ProfScope _prof("gather_x", st);
    const int64_t n = (s.T + 1) * B * 32;
    if (s.bf16)
      gather_x_kernel<__nv_bfloat16><<<grid_of(n), 256, 0, st>>>(
          s, B, (const __nv_bfloat16*)buf->x, buf->h0, buf->c0, idx,
          reinterpret_cast<__nv_bfloat16*>(wsb + L.xh), C);
    else
      gather_x_kernel<float><<<grid_of(n), 256, 0, st>>>(s, B, (const float*)buf->x, buf->h0,
                                                         buf->c0, idx,
                                                         reinterpret_cast<float*>(wsb + L.xh), C);
    PPO_LAUNCH_CHECK("gather_x_kernel");
  }
  ProfScope _prof("gather_rows", st);
  gather_rows_kernel<<<grid_of(s.T * B), 256, 0, st>>>(s, B, *buf, idx, act, head_on, avail,
                                                        logp_old, adv, ret, valid);
  PPO_LAUNCH_CHECK("gather_rows_kernel");
  return PPO_OK;
}

}  // extern "C"

// ============================================================================ NEXT-2
// Reward pipeline fused into the GAE load stage (App. Reward Weights P:1058-1079):
// game-time weighting of the shaped rewards (0.6^(T/10 min); win/loss exempt), team spirit
// r_i = (1-tau) rho_i + tau mean_team(rho), zero-sum (minus the enemy team's mean), division
// by the running reward std of the previous calls, then GAE.  One warp per game: a lane owns
// 8 consecutive steps of all 10 heroes (2 teams x 5), the 10 GAE recurrences are scanned
// across lanes together.  Per-block partial moments of the (unnormalised) final rewards are
// merged into the running statistics by reward_stats_kernel afterwards (fixed order).
namespace ppo {
namespace {

constexpr int kRewardBlocks = 148 * 4;

__device__ __forceinline__ void load8(const float* p, float (&v)[8]) {   // 32-byte aligned
  const float4 a = __ldcs(reinterpret_cast<const float4*>(p));
  const float4 b = __ldcs(reinterpret_cast<const float4*>(p) + 1);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void store8(float* p, const float (&v)[8]) {   // 32-byte aligned
  reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
  reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
}

__global__ void __launch_bounds__(128, 4) reward_gae_kernel(
    const float* __restrict__ shaped, const float* __restrict__ win,
    const int32_t* __restrict__ step0, int64_t G, int64_t L, const float* __restrict__ val,
    const uint8_t* __restrict__ done, ppo_reward_cfg cfg, const double* __restrict__ stats,
    float gamma, float lam, int seq_T, float* __restrict__ rew_out, float* __restrict__ adv,
    float* __restrict__ ret, double* __restrict__ partials, bool vec) {
  constexpr int NH = 10;
  __shared__ double red[4][3];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const double cnt = stats[0];
  const float inv_sigma = cnt > 0 ? (float)(1.0 / sqrt(fmax(stats[2] / cnt, 1e-16))) : 1.f;
  const float gl = gamma * lam;
  const float tau = cfg.tau;
  // 0.6^(T/10 min) = exp2(log2(0.6) * step * T_step / 600)
  const float dk = log2f(cfg.decay_base) * cfg.step_seconds / cfg.decay_seconds;
  const int64_t S = G * NH;
  const int64_t spr = seq_T > 0 ? L / seq_T : 0, nseq = S * spr;
  double ps = 0.0, pss = 0.0, pn = 0.0;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; g < G; g += nwarps) {
    float carry[NH];
#pragma unroll
    for (int i = 0; i < NH; ++i) carry[i] = 0.f;
    const int64_t s0 = g * NH;
    for (int64_t w_end = L; w_end > 0; w_end -= 256) {
      const int64_t w_start = w_end > 256 ? w_end - 256 : 0;
      const int64_t t0 = w_start + 8 * lane;
      const int n = (int)max((int64_t)0, min((int64_t)8, w_end - t0));
      // per step: decay, team means of the decayed raw rewards, GAE coefficient.  Full
      // chunks on a 32-byte grid (vec: L % 8 == 0 and aligned bases) load 16-byte vectors.
      const bool full = vec && n == 8;
      float cf[8], dec[8], mA[8], mB[8], nds[8];
      const float st0 = (float)step0[g];
      if (full) {
        const uint2 dw = __ldcs(reinterpret_cast<const uint2*>(done + g * L + t0));
        const uint8_t* db = reinterpret_cast<const uint8_t*>(&dw);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          nds[e] = db[e] ? 0.f : 1.f;
          cf[e] = gl * nds[e];
          dec[e] = exp2f(dk * (st0 + (float)(t0 + e)));
          mA[e] = 0.f;
          mB[e] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < NH; ++i) {
          float sh[8], wn[8];
          load8(shaped + (s0 + i) * L + t0, sh);
          load8(win + (s0 + i) * L + t0, wn);
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const float rho = sh[e] * dec[e] + wn[e];
            if (i < 5) mA[e] += rho;
            else mB[e] += rho;
          }
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          mA[e] *= 0.2f;
          mB[e] *= 0.2f;
        }
      } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const bool ok = e < n;
        const int64_t t = t0 + e;
        nds[e] = ok && !done[g * L + t] ? 1.f : 0.f;
        cf[e] = ok ? gl * nds[e] : 1.f;
        dec[e] = ok ? exp2f(dk * (st0 + (float)t)) : 0.f;
        float a = 0.f, b = 0.f;
        if (ok) {
#pragma unroll
          for (int i = 0; i < NH; ++i) {
            const float rho = shaped[(s0 + i) * L + t] * dec[e] + win[(s0 + i) * L + t];
            if (i < 5) a += rho;
            else b += rho;
          }
        }
        mA[e] = 0.2f * a;
        mB[e] = 0.2f * b;
      }
      }
#pragma unroll 1
      for (int i = 0; i < NH; ++i) {
        const float* vv = val + (s0 + i) * (L + 1);
        float delta[8], vk[9], sh[8], wn[8];
        if (full) {
          load8(shaped + (s0 + i) * L + t0, sh);
          load8(win + (s0 + i) * L + t0, wn);
          load_floats<9>(vv + t0, vk, val + S * (L + 1));
        }
        float rr[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const bool ok = e < n;
          const int64_t t = t0 + e;
          float dl = 0.f;
          if (ok) {
            const float rho = full ? sh[e] * dec[e] + wn[e]
                                   : shaped[(s0 + i) * L + t] * dec[e] + win[(s0 + i) * L + t];
            const float mt = i < 5 ? mA[e] : mB[e], me = i < 5 ? mB[e] : mA[e];
            float r = (1.f - tau) * rho + tau * mt;
            if (cfg.zero_sum) r -= me;
            ps += r;
            pss += (double)r * r;
            pn += 1.0;
            r *= inv_sigma;
            rr[e] = r;
            dl = full ? r + gamma * nds[e] * vk[e + 1] - vk[e]
                      : r + gamma * nds[e] * vv[t + 1] - vv[t];
          }
          delta[e] = dl;
        }
        if (rew_out) {
          if (full) {
            store8(rew_out + (s0 + i) * L + t0, rr);
          } else {
#pragma unroll
            for (int e = 0; e < 8; ++e)
              if (e < n) rew_out[(s0 + i) * L + t0 + e] = rr[e];
          }
        }
        float P = 0.f, Q = 1.f;
#pragma unroll
        for (int e = 7; e >= 0; --e) {
          P = delta[e] + cf[e] * P;
          Q = cf[e] * Q;
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
        const float a_first = P + Q * carry[i];
        float a = __shfl_down_sync(0xffffffffu, a_first, 1);
        if (lane == 31) a = carry[i];
        if (full && seq_T == 0) {
          float Ao[8], Ro[8];
#pragma unroll
          for (int e = 7; e >= 0; --e) {
            a = delta[e] + cf[e] * a;
            Ao[e] = a;
            Ro[e] = a + vk[e];
          }
          store8(adv + (s0 + i) * L + t0, Ao);
          store8(ret + (s0 + i) * L + t0, Ro);
        } else {
#pragma unroll
        for (int e = 7; e >= 0; --e) {
          if (e < n) {
            const int64_t t = t0 + e;
            a = delta[e] + cf[e] * a;
            int64_t o;
            if (seq_T > 0) {
              const int64_t k = t / seq_T, tt = t - k * seq_T;
              o = tt * nseq + (s0 + i) * spr + k;
            } else {
              o = (s0 + i) * L + t;
            }
            adv[o] = a;
            ret[o] = a + vv[t];
          }
        }
        }
        carry[i] = __shfl_sync(0xffffffffu, a_first, 0);
      }
    }
  }
  // deterministic partial moments: warp tree, then the block's 4 warps in order
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ps += __shfl_xor_sync(0xffffffffu, ps, o);
    pss += __shfl_xor_sync(0xffffffffu, pss, o);
    pn += __shfl_xor_sync(0xffffffffu, pn, o);
  }
  if (lane == 0) {
    red[wib][0] = pn;
    red[wib][1] = ps;
    red[wib][2] = pss;
  }
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0.0;
    for (int k = 0; k < 4; ++k) v += red[k][threadIdx.x];
    partials[blockIdx.x * 3 + threadIdx.x] = v;
  }
}

// Merge the batch moments into the running (count, mean, M2): Chan et al. pairwise update.
__global__ void reward_stats_kernel(const double* __restrict__ partials, int nblocks,
                                    double* __restrict__ stats) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double nb = 0.0, sb = 0.0, ssb = 0.0;
  for (int b = 0; b < nblocks; ++b) {
    nb += partials[3 * b];
    sb += partials[3 * b + 1];
    ssb += partials[3 * b + 2];
  }
  if (nb <= 0.0) return;
  const double mb = sb / nb;
  const double m2b = fmax(ssb - nb * mb * mb, 0.0);
  const double n0 = stats[0], mean0 = stats[1], m20 = stats[2];
  const double n = n0 + nb;
  const double d = mb - mean0;
  stats[0] = n;
  stats[1] = mean0 + d * nb / n;
  stats[2] = m20 + m2b + d * d * n0 * nb / n;
}

}  // namespace
}  // namespace ppo

extern "C" {

int ppo_reward_gae_scratch_bytes(size_t* bytes) {
  if (!bytes) return fail(PPO_E_ARG, "bytes is NULL");
  *bytes = sizeof(double) * 3 * kRewardBlocks;
  return PPO_OK;
}

int ppo_reward_gae(const float* shaped, const float* win, const int32_t* step0, int64_t G,
                   int64_t L, const float* val, const uint8_t* done, const ppo_reward_cfg* cfg,
                   double* stats, float gamma, float lam, int32_t seq_T, float* rew_out,
                   float* adv, float* ret, void* scratch, size_t scratch_bytes,
                   ppo_stream_t st_) {
  cudaStream_t st = (cudaStream_t)st_;
  if (G < 0 || L < 0) return fail(PPO_E_SHAPE, "G and L must be >= 0");
  if (G == 0 || L == 0) return PPO_OK;
  if (!shaped || !win || !step0 || !val || !done || !cfg || !stats || !adv || !ret)
    return fail(PPO_E_ARG, "NULL pointer");
  if (seq_T < 0 || (seq_T > 0 && L % seq_T)) return fail(PPO_E_SHAPE, "L must be a multiple of seq_T");
  if (!scratch || scratch_bytes < sizeof(double) * 3 * kRewardBlocks || !aligned(scratch, 8))
    return fail(PPO_E_ARG, "scratch too small (ppo_reward_gae_scratch_bytes)");
  if (!(cfg->tau >= 0.f && cfg->tau <= 1.f) || !(cfg->decay_base > 0.f) ||
      !(cfg->decay_seconds > 0.f) || !(cfg->step_seconds > 0.f))
    return fail(PPO_E_ARG, "bad reward config");
  double* partials = static_cast<double*>(scratch);
  {
    ProfScope _prof("reward_gae", st);
    // 16-byte vectors for full 8-step chunks: L % 8 == 0 and 32-byte aligned bases
    const bool vec = L % 8 == 0 && aligned(shaped, 32) && aligned(win, 32) && aligned(done, 8) &&
                     aligned(adv, 32) && aligned(ret, 32) && (!rew_out || aligned(rew_out, 32));
    reward_gae_kernel<<<kRewardBlocks, 128, 0, st>>>(shaped, win, step0, G, L, val, done, *cfg,
                                                     stats, gamma, lam, seq_T, rew_out, adv, ret,
                                                     partials, vec);
    PPO_LAUNCH_CHECK("reward_gae_kernel");
  }
  ProfScope _prof("reward_stats", st);
  reward_stats_kernel<<<1, 32, 0, st>>>(partials, kRewardBlocks, stats);
  PPO_LAUNCH_CHECK("reward_stats_kernel");
  return PPO_OK;
}

}  // extern "C"
