// comm.cu -- a9: data-parallel gradient average ("Gradients are averaged across the
// pool using NCCL2 allreduce before being synchronously applied").  libppo5 owns its NCCL
// communicator; the unique id travels over the caller's torch process group.
#include <cuda.h>
#include <cuda_bf16.h>
#include <nccl.h>

#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

// a9+a10 over NVLink peer memory (SURVEY §8(e) option): the buffers every rank's fused
// kernel reads or writes on its peers, mapped through CUDA IPC by ppo_dp_attach.
struct DpPeers {
  const float* g[PPO_DP_MAX_RANKS];
  float* p[PPO_DP_MAX_RANKS];
  __nv_bfloat16* pb[PPO_DP_MAX_RANKS];
};

struct ppo_comm {
  ncclComm_t comm;
  int rank, world;
  // ppo_dp_attach state
  bool attached = false;
  size_t n = 0;
  DpPeers peers{};
  std::vector<void*> mapped;   // IPC mappings to close
  float* sync = nullptr;       // 1-float device scratch for the stream-ordered barriers
  float* stage = nullptr;      // push mode: world x shard floats, slot j = rank j's gradient
  ppo::DpStage dst{};          // every rank's staging, as the backward's epilogues see it
};

namespace {
int nccl_fail(ncclResult_t r, const char* what) {
  return ppo::fail(PPO_E_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}
}  // namespace

extern "C" {

int ppo_comm_unique_id(uint8_t id[PPO_COMM_ID_BYTES]) {
  static_assert(sizeof(ncclUniqueId) == PPO_COMM_ID_BYTES, "ncclUniqueId size");
  if (!id) return ppo::fail(PPO_E_ARG, "id is NULL");
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
  memcpy(id, &u, sizeof(u));
  return PPO_OK;
}

int ppo_comm_init(const uint8_t id[PPO_COMM_ID_BYTES], int rank, int world, ppo_comm** out) {
  if (!id || !out) return ppo::fail(PPO_E_ARG, "NULL pointer");
  if (world < 1 || rank < 0 || rank >= world) return ppo::fail(PPO_E_ARG, "bad rank/world");
  ncclUniqueId u;
  memcpy(&u, id, sizeof(u));
  ppo_comm* c = new ppo_comm{nullptr, rank, world};
  ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return nccl_fail(r, "ncclCommInitRank");
  }
  *out = c;
  return PPO_OK;
}

int grad_allreduce(ppo_comm* c, float* g, size_t n, int32_t n_buckets, ppo_stream_t st) {
  if (!c) return ppo::fail(PPO_E_ARG, "comm is NULL");
  if (n == 0 || c->world == 1) return PPO_OK;
  if (!g) return ppo::fail(PPO_E_ARG, "g is NULL");
  if (n_buckets <= 0) n_buckets = 1;
  const size_t per = (n + n_buckets - 1) / n_buckets;
  ppo::ProfScope _prof("allreduce", (cudaStream_t)st);
  ncclResult_t r = ncclGroupStart();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
  for (size_t off = 0; off < n; off += per) {
    const size_t cnt = off + per <= n ? per : n - off;
    r = ncclAllReduce(g + off, g + off, cnt, ncclFloat32, ncclAvg, c->comm, (cudaStream_t)st);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return nccl_fail(r, "ncclAllReduce");
    }
  }
  r = ncclGroupEnd();
  if (r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
  return PPO_OK;
}

int ppo_comm_destroy(ppo_comm* c) {
  if (!c) return PPO_OK;
  for (void* m : c->mapped) cudaIpcCloseMemHandle(m);
  if (c->sync) cudaFree(c->sync);
  if (c->stage) cudaFree(c->stage);
  ncclResult_t r = ncclCommDestroy(c->comm);
  delete c;
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return PPO_OK;
}

}  // extern "C"

// the push-mode staging map of an attached comm with world > 1 (NULL otherwise); api.cu
const ppo::DpStage* ppo_comm_dp_stage(const ppo_comm* c) {
  return c && c->attached && c->world > 1 ? &c->dst : nullptr;
}
size_t ppo_comm_dp_n(const ppo_comm* c) { return c ? c->n : 0; }

extern "C" {

size_t ppo_dp_shard(size_t n, int world) {
  if (world < 1) return 0;
  const size_t per = (n + (size_t)world - 1) / (size_t)world;
  return (per + 63) / 64 * 64;
}

namespace {
using GetRangeFn = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);

// base of the allocation holding ptr (IPC handles name whole cudaMalloc allocations)
int alloc_base(const void* ptr, char** base) {
  static GetRangeFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    PPO_CUDA_CHECK(cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &f, 12000,
                                                    cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f)
      return ppo::fail(PPO_E_CUDA, "cuMemGetAddressRange entry point not found");
    fn = reinterpret_cast<GetRangeFn>(f);
  }
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return ppo::fail(PPO_E_ARG, "pointer is not device memory from cudaMalloc");
  *base = reinterpret_cast<char*>(b);
  return PPO_OK;
}

struct IpcRecord {          // what one rank publishes for one buffer
  cudaIpcMemHandle_t h;
  uint64_t off;
  uint64_t present;
};

// a9 + a10 on the rank's shard: peers' grads in, the updated shard out to every rank
// stage (push mode, nullable): the owner's staging, slot j = rank j's gradient of the shard
// (written by the backward's epilogues); else (pull mode) the peers' gradients over NVLink
__global__ void __launch_bounds__(256) dp_adam_kernel(DpPeers pe, int world, int rank,
                                                      size_t lo, size_t hi, float* __restrict__ m,
                                                      float* __restrict__ v, ppo::AdamParams ap,
                                                      float inv_world,
                                                      const float* __restrict__ stage,
                                                      size_t shard, size_t shard_lo) {
  auto gsrc = [&](int j, size_t e) -> const float* {   // rank j's gradient element e
    return stage ? stage + (size_t)j * shard + (e - shard_lo) : pe.g[j] + e;
  };
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t lo4 = lo / 4, hi4 = hi / 4;           // lo is a multiple of 64
  for (size_t i = lo4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < hi4; i += stride) {
    // g = (1/N) sum over ranks in rank order: the same bits on every rank's shard owner
    float4 gs = *reinterpret_cast<const float4*>(gsrc(0, 4 * i));
    for (int j = 1; j < world; ++j) {
      const float4 gj = *reinterpret_cast<const float4*>(gsrc(j, 4 * i));
      gs.x += gj.x;
      gs.y += gj.y;
      gs.z += gj.z;
      gs.w += gj.w;
    }
    float4 pp = reinterpret_cast<const float4*>(pe.p[rank])[i];
    float4 mm = reinterpret_cast<float4*>(m)[i];
    float4 vv = reinterpret_cast<float4*>(v)[i];
    ppo::adam_elem(ap, __fmul_rn(gs.x, inv_world), pp.x, mm.x, vv.x);
    ppo::adam_elem(ap, __fmul_rn(gs.y, inv_world), pp.y, mm.y, vv.y);
    ppo::adam_elem(ap, __fmul_rn(gs.z, inv_world), pp.z, mm.z, vv.z);
    ppo::adam_elem(ap, __fmul_rn(gs.w, inv_world), pp.w, mm.w, vv.w);
    reinterpret_cast<float4*>(m)[i] = mm;
    reinterpret_cast<float4*>(v)[i] = vv;
    uint2 u;
    if (pe.pb[rank]) {
      __nv_bfloat162 a = __floats2bfloat162_rn(pp.x, pp.y), b = __floats2bfloat162_rn(pp.z, pp.w);
      u.x = *reinterpret_cast<uint32_t*>(&a);
      u.y = *reinterpret_cast<uint32_t*>(&b);
    }
    // all-gather over NVLink of what the forward reads: the bf16 shadow when there is one
    // (theta then stays sharded like m, v), else theta itself
    if (pe.pb[rank]) {
      reinterpret_cast<float4*>(pe.p[rank])[i] = pp;
      for (int j = 0; j < world; ++j) reinterpret_cast<uint2*>(pe.pb[j])[i] = u;
    } else {
      for (int j = 0; j < world; ++j) reinterpret_cast<float4*>(pe.p[j])[i] = pp;
    }
  }
  // scalar tail (n % 4) on the last shard
  for (size_t i = hi4 * 4 + blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < hi; i += stride) {
    float gi = *gsrc(0, i);
    for (int j = 1; j < world; ++j) gi += *gsrc(j, i);
    float pi = pe.p[rank][i], mi = m[i], vi = v[i];
    ppo::adam_elem(ap, __fmul_rn(gi, inv_world), pi, mi, vi);
    m[i] = mi;
    v[i] = vi;
    if (pe.pb[rank]) {
      pe.p[rank][i] = pi;
      for (int j = 0; j < world; ++j) pe.pb[j][i] = __float2bfloat16_rn(pi);
    } else {
      for (int j = 0; j < world; ++j) pe.p[j][i] = pi;
    }
  }
  __threadfence_system();
}

int launch_dp_adam(const DpPeers& pe, int world, int rank, size_t lo, size_t hi, float* m,
                   float* v, const ppo::AdamParams& ap, const float* stage, size_t shard,
                   cudaStream_t st, size_t shard_lo) {
  ppo::ProfScope _prof("dp_adam", st);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const size_t units = (hi - lo) / 4 + 1;
  const int grid = (int)std::min<size_t>((size_t)sms * 8, (units + 255) / 256);
  dp_adam_kernel<<<std::max(grid, 1), 256, 0, st>>>(pe, world, rank, lo, hi, m, v, ap,
                                                    1.0f / (float)world, stage, shard, shard_lo);
  PPO_LAUNCH_CHECK("dp_adam_kernel");
  return PPO_OK;
}

int barrier(ppo_comm* c, cudaStream_t st) {   // stream-ordered: a 1-float NCCL allreduce
  ncclResult_t r = ncclAllReduce(c->sync, c->sync, 1, ncclFloat32, ncclSum, c->comm, st);
  return r == ncclSuccess ? PPO_OK : nccl_fail(r, "ncclAllReduce (barrier)");
}
}  // namespace

int ppo_dp_attach(ppo_comm* c, float* g, float* p, uint16_t* p_bf16, size_t n) {
  if (!c) return ppo::fail(PPO_E_ARG, "comm is NULL");
  if (!g || !p) return ppo::fail(PPO_E_ARG, "g or p is NULL");
  if (c->attached) return ppo::fail(PPO_E_ARG, "buffers already attached to this comm");
  if (c->world > PPO_DP_MAX_RANKS) return ppo::fail(PPO_E_SHAPE, "world exceeds PPO_DP_MAX_RANKS");
  if (!ppo::aligned(g, 16) || !ppo::aligned(p, 16) || (p_bf16 && !ppo::aligned(p_bf16, 16)))
    return ppo::fail(PPO_E_ALIGN, "dp buffers must be 16-byte aligned");
  const int W = c->world;
  const size_t sh = ppo_dp_shard(n, W);
  // push-mode staging, owned by the comm (the backward's epilogues write into the owners')
  if (W > 1) PPO_CUDA_CHECK(cudaMalloc(&c->stage, (size_t)W * sh * sizeof(float)));
  void* bufs[4] = {g, p, p_bf16, c->stage};
  IpcRecord mine[4];
  memset(mine, 0, sizeof(mine));
  for (int k = 0; k < 4; ++k) {
    if (!bufs[k] || W == 1) continue;
    char* base = nullptr;
    int rc = alloc_base(bufs[k], &base);
    if (rc != PPO_OK) return rc;
    PPO_CUDA_CHECK(cudaIpcGetMemHandle(&mine[k].h, base));
    mine[k].off = (uint64_t)(static_cast<char*>(bufs[k]) - base);
    mine[k].present = 1;
  }
  // all-gather the records over NCCL (device staging, synchronous)
  const size_t rec = sizeof(mine);
  std::vector<uint8_t> all(rec * W);
  if (W > 1) {
    uint8_t* dbuf = nullptr;
    cudaStream_t st;
    PPO_CUDA_CHECK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    PPO_CUDA_CHECK(cudaMalloc(&dbuf, rec * W));
    PPO_CUDA_CHECK(cudaMemcpyAsync(dbuf + rec * c->rank, mine, rec, cudaMemcpyHostToDevice, st));
    ncclResult_t r = ncclAllGather(dbuf + rec * c->rank, dbuf, rec, ncclUint8, c->comm, st);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllGather (ipc handles)");
    PPO_CUDA_CHECK(cudaMemcpyAsync(all.data(), dbuf, rec * W, cudaMemcpyDeviceToHost, st));
    PPO_CUDA_CHECK(cudaStreamSynchronize(st));
    PPO_CUDA_CHECK(cudaFree(dbuf));
    PPO_CUDA_CHECK(cudaStreamDestroy(st));
  }
  DpPeers pe{};
  ppo::DpStage ds{};
  ds.world = W;
  ds.rank = c->rank;
  ds.shard = (int64_t)sh;
  for (int j = 0; j < W; ++j) {
    if (j == c->rank) {
      pe.g[j] = g;
      pe.p[j] = p;
      pe.pb[j] = reinterpret_cast<__nv_bfloat16*>(p_bf16);
      ds.stage[j] = c->stage;
      continue;
    }
    const IpcRecord* r = reinterpret_cast<const IpcRecord*>(all.data() + rec * j);
    char* mapped[4] = {nullptr, nullptr, nullptr, nullptr};
    for (int k = 0; k < 4; ++k) {
      if (!r[k].present) continue;
      // one mapping per distinct allocation of rank j
      for (int q = 0; q < k && !mapped[k]; ++q)
        if (r[q].present && !memcmp(&r[q].h, &r[k].h, sizeof(r[k].h)))
          mapped[k] = mapped[q] - r[q].off;
      if (!mapped[k]) {
        void* m = nullptr;
        PPO_CUDA_CHECK(cudaIpcOpenMemHandle(&m, r[k].h, cudaIpcMemLazyEnablePeerAccess));
        c->mapped.push_back(m);
        mapped[k] = static_cast<char*>(m);
      }
      mapped[k] += r[k].off;
    }
    pe.g[j] = reinterpret_cast<const float*>(mapped[0]);
    pe.p[j] = reinterpret_cast<float*>(mapped[1]);
    pe.pb[j] = reinterpret_cast<__nv_bfloat16*>(mapped[2]);
    ds.stage[j] = reinterpret_cast<float*>(mapped[3]);
    if (!pe.g[j] || !pe.p[j] || (p_bf16 && !pe.pb[j]) || !ds.stage[j])
      return ppo::fail(PPO_E_ARG, "ranks disagree on which dp buffers exist");
  }
  if (!c->sync) PPO_CUDA_CHECK(cudaMalloc(&c->sync, 16));
  PPO_CUDA_CHECK(cudaMemset(c->sync, 0, 16));
  c->peers = pe;
  c->dst = W > 1 ? ds : ppo::DpStage{};
  c->n = n;
  c->attached = true;
  return PPO_OK;
}

int ppo_dp_adam_step(ppo_comm* c, float* m, float* v, int64_t t, double lr, double b1,
                     double b2, double eps, double clip_sigma, int32_t staged, ppo_stream_t s) {
  if (!c) return ppo::fail(PPO_E_ARG, "comm is NULL");
  return ppo_dp_adam_step_range(c, m, v, t, lr, b1, b2, eps, clip_sigma, staged, 0, c->n, s);
}

int ppo_dp_adam_step_range(ppo_comm* c, float* m, float* v, int64_t t, double lr, double b1,
                           double b2, double eps, double clip_sigma, int32_t staged,
                           size_t range_lo, size_t range_hi, ppo_stream_t s) {
  if (!c) return ppo::fail(PPO_E_ARG, "comm is NULL");
  if (!c->attached) return ppo::fail(PPO_E_ARG, "ppo_dp_attach was not called on this comm");
  if (!m || !v) return ppo::fail(PPO_E_ARG, "m or v is NULL");
  if (!ppo::aligned(m, 16) || !ppo::aligned(v, 16))
    return ppo::fail(PPO_E_ALIGN, "m and v must be 16-byte aligned");
  if (t < 1) return ppo::fail(PPO_E_ARG, "t must be >= 1");
  if (!(b1 >= 0.0 && b1 < 1.0 && b2 >= 0.0 && b2 < 1.0)) return ppo::fail(PPO_E_ARG, "bad betas");
  const ppo::AdamParams ap = ppo::make_adam_params(t, lr, b1, b2, eps, clip_sigma);
  if (range_lo > range_hi || range_hi > c->n || (range_lo % 64) ||
      (range_hi % 64 && range_hi != c->n))
    return ppo::fail(PPO_E_ARG, "range must be [lo, hi) within theta, multiples of 64 (or hi = n)");
  const size_t sh = ppo_dp_shard(c->n, c->world);
  const size_t slo = std::min(c->n, sh * (size_t)c->rank), shi = std::min(c->n, slo + sh);
  // this rank's shard within the range (possibly empty; the barriers still run)
  const size_t lo = std::max(slo, range_lo), hi = std::max(lo, std::min(shi, range_hi));
  cudaStream_t st = (cudaStream_t)s;
  int rc = PPO_OK;
  if (c->world > 1 && (rc = barrier(c, st)) != PPO_OK) return rc;   // every grad is final
  rc = launch_dp_adam(c->peers, c->world, c->rank, lo, hi, m, v, ap,
                      staged && c->world > 1 ? c->stage : nullptr, sh, st, slo);
  if (rc != PPO_OK) return rc;
  // every rank's writes into this rank's theta/shadow have landed, and no rank still reads
  // this rank's grad, before the caller's next step
  if (c->world > 1 && (rc = barrier(c, st)) != PPO_OK) return rc;
  return PPO_OK;
}

int ppo_dp_allgather(ppo_comm* c, float* buf, ppo_stream_t s) {
  if (!c) return ppo::fail(PPO_E_ARG, "comm is NULL");
  if (!c->attached) return ppo::fail(PPO_E_ARG, "ppo_dp_attach was not called on this comm");
  if (!buf) return ppo::fail(PPO_E_ARG, "buf is NULL");
  if (c->world == 1) return PPO_OK;
  const size_t sh = ppo_dp_shard(c->n, c->world);
  ncclResult_t r = ncclAllGather(buf + sh * (size_t)c->rank, buf, sh, ncclFloat32, c->comm,
                                 (cudaStream_t)s);
  return r == ncclSuccess ? PPO_OK : nccl_fail(r, "ncclAllGather");
}

int ppo_test_dp_adam(int32_t world, const float* const* g, float* const* p,
                     uint16_t* const* p_bf16, float* const* m, float* const* v,
                     const float* const* stage, size_t n, int64_t t, double lr, double b1,
                     double b2, double eps, double clip_sigma, ppo_stream_t s) {
  if (world < 1 || world > PPO_DP_MAX_RANKS) return ppo::fail(PPO_E_ARG, "world out of range");
  if (!g || !p || !m || !v) return ppo::fail(PPO_E_ARG, "NULL pointer array");
  if (t < 1) return ppo::fail(PPO_E_ARG, "t must be >= 1");
  if (!(b1 >= 0.0 && b1 < 1.0 && b2 >= 0.0 && b2 < 1.0)) return ppo::fail(PPO_E_ARG, "bad betas");
  if (n == 0) return PPO_OK;
  DpPeers pe{};
  const bool shadow = p_bf16 && p_bf16[0];
  for (int j = 0; j < world; ++j) {
    if (!g[j] || !p[j] || !m[j] || !v[j] || (shadow && !p_bf16[j]) || (stage && !stage[j]))
      return ppo::fail(PPO_E_ARG, "NULL buffer of a virtual rank");
    if (!ppo::aligned(g[j], 16) || !ppo::aligned(p[j], 16) || !ppo::aligned(m[j], 16) ||
        !ppo::aligned(v[j], 16) || (shadow && !ppo::aligned(p_bf16[j], 16)) ||
        (stage && !ppo::aligned(stage[j], 16)))
      return ppo::fail(PPO_E_ALIGN, "dp buffers must be 16-byte aligned");
    pe.g[j] = g[j];
    pe.p[j] = p[j];
    pe.pb[j] = shadow ? reinterpret_cast<__nv_bfloat16*>(p_bf16[j]) : nullptr;
  }
  const ppo::AdamParams ap = ppo::make_adam_params(t, lr, b1, b2, eps, clip_sigma);
  const size_t sh = ppo_dp_shard(n, world);
  // every virtual rank's launch, in rank order on one stream: the stream order stands in for
  // the two NCCL barriers of ppo_dp_adam_step (all gradients final before, all peer stores
  // landed after)
  for (int r = 0; r < world; ++r) {
    const size_t lo = std::min(n, sh * (size_t)r), hi = std::min(n, lo + sh);
    if (lo == hi) continue;
    const int rc = launch_dp_adam(pe, world, r, lo, hi, m[r], v[r], ap,
                                  stage && world > 1 ? stage[r] : nullptr, sh, (cudaStream_t)s, lo);
    if (rc != PPO_OK) return rc;
  }
  return PPO_OK;
}

}  // extern "C"
