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
