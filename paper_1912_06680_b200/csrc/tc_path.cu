// tc_path.cu -- the bf16 tcgen05 path of the step: TMA tensor maps over the workspace and
// the GEMM launches for forward (a2-a4) and backward (a6-a8).  DESIGN.md "Data layout".
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "tc_gemm.cuh"

namespace ppo {
namespace {

// Tile-scheduler counters of the standalone test GEMM (ppo_test_tc_gemm, tests only); the
// step's GEMMs use the counters in their workspace (common.cuh SchedSlot).
__device__ unsigned int g_test_sched_ctr[kSchedWords];

unsigned int* test_sched_counter() {
  static unsigned int* base[64] = {nullptr};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  if (!base[dev]) {
    void* p = nullptr;
    if (cudaGetSymbolAddress(&p, g_test_sched_ctr) != cudaSuccess) return nullptr;
    base[dev] = static_cast<unsigned int*>(p);
  }
  return base[dev];
}

// ---- SM -> die map (B200: 2 dies; every 2 KB of address space is homed on one of them, and an
// SM reads a line homed on its own die ~70 cycles faster).  Probe: each SM times chains of
// dependent L2 hits on kDieLines lines 2 KB apart; per line the SMs split into a fast and a
// slow group, and each SM's pattern over the lines correlates +-1 with a reference SM's.
constexpr int kDieLines = 64, kDieReps = 24, kDieMaxSm = 256;
__global__ void die_probe_kernel(const unsigned* buf, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  unsigned v = 0;
  const uint32_t sm = tc::smid();
  for (int l = 0; l < kDieLines; ++l) {
    const unsigned* a = buf + (size_t)l * 512;
    asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(a + v));
    const long long t0 = clock64();
    for (int r = 0; r < kDieReps; ++r)
      asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(v) : "l"(a + v));
    const long long t1 = clock64();
    out[(size_t)blockIdx.x * kDieLines + l] =
        (unsigned long long)(t1 - t0) | ((unsigned long long)sm << 48);
  }
  if (v == 0xFFFFFFFFu) out[0] = 0;   // keep the chain live (buf is zero)
}

struct DieMap {
  uint8_t* dev = nullptr;
  int n0 = 0, n1 = 0;
  bool done = false;
};

int probe_die_map(DieMap& dm) {
  int sms = num_sms();
  if (sms > kDieMaxSm) return PPO_E_UNSUPPORTED;
  const int nb = 4 * sms;
  unsigned* buf = nullptr;
  unsigned long long* out = nullptr;
  PPO_CUDA_CHECK(cudaMalloc(&buf, (size_t)kDieLines * 2048));
  PPO_CUDA_CHECK(cudaMalloc(&out, (size_t)nb * kDieLines * 8));
  PPO_CUDA_CHECK(cudaMemset(buf, 0, (size_t)kDieLines * 2048));
  for (int rep = 0; rep < 2; ++rep) die_probe_kernel<<<nb, 32>>>(buf, out);
  std::vector<unsigned long long> h((size_t)nb * kDieLines);
  const cudaError_t e = cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  cudaFree(out);
  if (e != cudaSuccess) return fail(PPO_E_CUDA, cudaGetErrorString(e));
  std::vector<double> lat((size_t)sms * kDieLines, 0.0);
  std::vector<int> cnt(sms, 0);
  for (int b = 0; b < nb; ++b) {
    const int sm = (int)(h[(size_t)b * kDieLines] >> 48);
    if (sm < 0 || sm >= sms) continue;
    ++cnt[sm];
    for (int l = 0; l < kDieLines; ++l)
      lat[(size_t)sm * kDieLines + l] += (double)(h[(size_t)b * kDieLines + l] & 0xFFFFFFFFFFFFull);
  }
  // per line: SMs faster than the midpoint of the line's fastest and slowest SM are on the
  // line's home die; align every line's split to line 0's (a line homed on the other die
  // flips it) and give each SM its majority.  A misassigned SM costs locality, not results.
  std::vector<int> votes(sms, 0), ref;
  double gap = 0.0;
  for (int l = 0; l < kDieLines; ++l) {
    double lo = 1e30, hi = 0.0;
    for (int s = 0; s < sms; ++s) {
      if (!cnt[s]) continue;
      const double x = lat[(size_t)s * kDieLines + l] / cnt[s];
      lo = std::min(lo, x);
      hi = std::max(hi, x);
    }
    gap += (hi - lo) / kDieReps / kDieLines;
    const double mid = 0.5 * (lo + hi);
    std::vector<int> fast(sms, 0);
    for (int s = 0; s < sms; ++s) fast[s] = cnt[s] && lat[(size_t)s * kDieLines + l] / cnt[s] < mid;
    if (ref.empty()) ref = fast;
    int agree = 0;
    for (int s = 0; s < sms; ++s) agree += fast[s] == ref[s];
    const bool flip = 2 * agree < sms;
    for (int s = 0; s < sms; ++s) votes[s] += (fast[s] ^ (int)flip) ? 1 : -1;
  }
  if (gap < 20.0) return PPO_E_UNSUPPORTED;   // no near/far split (one die)
  std::vector<uint8_t> die(sms, 0);
  int n0 = 0;
  for (int s = 0; s < sms; ++s) {
    die[s] = votes[s] > 0 ? 0 : 1;
    n0 += die[s] == 0;
  }
  if (n0 < sms / 4 || n0 > sms - sms / 4) return PPO_E_UNSUPPORTED;
  PPO_CUDA_CHECK(cudaMalloc(&dm.dev, kDieMaxSm));
  PPO_CUDA_CHECK(cudaMemset(dm.dev, 0, kDieMaxSm));
  PPO_CUDA_CHECK(cudaMemcpy(dm.dev, die.data(), sms, cudaMemcpyHostToDevice));
  dm.n0 = n0;
  dm.n1 = sms - n0;
  return PPO_OK;
}

// Die-aware tile queues for the CTA-pair GEMMs: off.  Measured (profiles/r02_ab_die_sched2.txt,
// same box, interleaved): each die taking a contiguous half of the raster made the step 7%
// slower -- DRAM reads of the backward step GEMM rose from 9.6 to 14 GB per launch and the
// cross-die (ltcfabric) traffic by 27%: both dies then stream the shared operand panels
// separately.  PPO_DIE_SCHED=1 re-enables it in experiment builds.
bool die_sched() { return knob_int("PPO_DIE_SCHED", 0) != 0; }

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 3-D bf16 tensor map, dims innermost first; strides in bytes for dims 1 and 2.
int make_map(CUtensorMap* m, const void* base, uint64_t d0, uint64_t d1, uint64_t d2,
             uint64_t s1, uint64_t s2, uint32_t box0, uint32_t box1) {
  auto fn = encode_fn();
  if (!fn) return fail(PPO_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (d2 == 1) s2 = s1 * d1;
  const cuuint64_t dims[3] = {d0, d1, d2};
  const cuuint64_t strides[2] = {s1, s2};
  const cuuint32_t box[3] = {box0, box1, 1};
  const cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(PPO_E_CUDA, "cuTensorMapEncodeTiled failed (code " + std::to_string((int)r) +
                                 ") d0=" + std::to_string(d0) + " d1=" + std::to_string(d1));
  return PPO_OK;
}

// K-major operand [rows][K] (K contiguous): box {64, tile rows}.
int map_kmajor(CUtensorMap* m, const void* base, uint64_t K, uint64_t rows, uint64_t ld_elems,
               uint64_t Z, uint64_t zstride_elems, uint32_t box_rows) {
  return make_map(m, base, K, rows, Z, ld_elems * 2, zstride_elems * 2, 64, box_rows);
}
// MN-major operand [K][MN] (MN contiguous): box {64 (MN panel), 64 (K)}.
int map_mnmajor(CUtensorMap* m, const void* base, uint64_t MN, uint64_t K, uint64_t ld_elems) {
  return make_map(m, base, MN, K, 1, ld_elems * 2, 0, 64, tc::BK);
}

// Row-interleaved K-major view for single-tile multi-step launches (TileShape::a_ilv):
// dims {K, rows / 4 (i), 4 (q), Z} with strides {4 ld, ld, zstride}: a {64, 32, 4, 1} box puts
// row 4 i + q of a 128-row block at smem row 32 q + i.
int map_kmajor_ilv(CUtensorMap* m, const void* base, uint64_t K, uint64_t rows, uint64_t ld_elems,
                   uint64_t Z, uint64_t zstride_elems) {
  auto fn = encode_fn();
  if (!fn) return fail(PPO_E_CUDA, "cuTensorMapEncodeTiled unavailable");
  if (rows % 4 != 0) return fail(PPO_E_SHAPE, "interleaved map needs rows % 4 == 0");
  const cuuint64_t dims[4] = {K, rows / 4, 4, Z};
  const cuuint64_t strides[3] = {4 * ld_elems * 2, ld_elems * 2,
                                 (Z > 1 ? zstride_elems : rows * ld_elems) * 2};
  const cuuint32_t box[4] = {64, 32, 4, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(PPO_E_CUDA, "cuTensorMapEncodeTiled (interleaved) failed (code " +
                                std::to_string((int)r) + ")");
  return PPO_OK;
}
// Single 256-row tile per step (B <= 256, B % 4 == 0): interleave the rows over the four TMEM
// lane quarters so a small batch's epilogue runs on all four epilogue warps (the backward's:
// tiny config 311 -> 287 us, profiles/r02_ilv_tiny.txt).  PPO_ILV=0 (experiment builds) keeps
// the natural order.
bool use_ilv(int64_t B) { return B <= 256 && B % 4 == 0 && knob_int("PPO_ILV", 1) != 0; }

template <int BN, bool A_MN, bool B_MN, class Epi, int STAGES = 4>
int launch(const char* tag, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0,
           const CUtensorMap& b1, const tc::TileShape& sh, const Epi& epi, cudaStream_t st,
           bool pdl = false) {
  using L = tc::Smem<BN, A_MN, B_MN, STAGES>;
  auto kern = tc::tc_gemm_kernel<BN, A_MN, B_MN, STAGES, Epi>;
  static bool configured = false;
  if (!configured) {
    PPO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL));
    configured = true;
  }
  if (sh.nkb0 + sh.nkb1 <= 0) return fail(PPO_E_SHAPE, "GEMM with empty K");
  if (!sh.sched) return fail(PPO_E_CUDA, "tile scheduler counter unavailable");
  const int64_t ntiles = (int64_t)((sh.M + tc::BM - 1) / tc::BM) * ((sh.N + BN - 1) / BN);
  const bool all_tiles = knob_int("PPO_GRID_ALL_TILES", 0) != 0;
  const int grid = (int)std::min<int64_t>(ntiles * std::max(sh.ksplit, 1),
                                          all_tiles ? (int64_t)1 << 30 : num_sms());
  if (grid <= 0) return PPO_OK;
  ProfScope _prof(tag, st);
  if (pdl) {
    PPO_CUDA_CHECK(launch_pdl(kern, dim3(grid), dim3(tc::kThreads), L::TOTAL, st, a0, a1, b0,
                              b1, sh, epi));
  } else {
    kern<<<grid, tc::kThreads, L::TOTAL, st>>>(a0, a1, b0, b1, sh, epi);
  }
  PPO_LAUNCH_CHECK("tc_gemm_kernel");
  return PPO_OK;
}

// CTA-pair launch: 256x256 tiles, grid = 2 x clusters (one CTA per SM, persistent).
template <bool A_MN, bool B_MN, class Epi, int MB = 1, int BN = 256, bool MS = false>
int launch2(const char* tag, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0,
            const CUtensorMap& b1, const tc::TileShape& sh, const Epi& epi, cudaStream_t st) {
  constexpr int STAGES = MB == 1 ? 6 : 4;
  using L = tc::Smem2<A_MN, B_MN, STAGES, MB, BN>;
  auto kern = tc::tc_gemm2_kernel<A_MN, B_MN, STAGES, MB, BN, Epi, MS>;
  if ((sh.tsteps > 1) != MS) return fail(PPO_E_SHAPE, "multi-step launch without the MS kernel");
  static bool configured = false;
  if (!configured) {
    PPO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL));
    configured = true;
  }
  if (sh.nkb0 + sh.nkb1 <= 0) return fail(PPO_E_SHAPE, "GEMM with empty K");
  if (!sh.sched) return fail(PPO_E_CUDA, "tile scheduler counter unavailable");
  const int64_t ntiles = (int64_t)((sh.M + 256 * MB - 1) / (256 * MB)) * ((sh.N + BN - 1) / BN) *
                         std::max(sh.ksplit, 1);
  // PPO_GRID_ALL_TILES=1 (or PPO_GRID_ALL_TILES_<tag>=1): one cluster per tile, hardware-
  // ordered dispatch instead of the persistent schedule (experiment knob)
  bool all_tiles = knob_int("PPO_GRID_ALL_TILES", 0) != 0;
#ifdef PPO_EXPERIMENTS
  {
    char n[64];
    snprintf(n, sizeof(n), "PPO_GRID_ALL_TILES_%s", tag);
    all_tiles = all_tiles || knob_int(n, 0) != 0;
  }
#endif
  const int clusters = (int)std::min<int64_t>(ntiles, all_tiles ? (int64_t)1 << 30 : num_sms() / 2);
  if (clusters <= 0) return PPO_OK;
  tc::TileShape shd = sh;
  if (die_sched()) {
    // die-aware queues: each die gets a share of the raster sequence proportional to the CTA
    // pairs it hosts (clusters are placed within one die)
    int n0 = 0, n1 = 0;
    const uint8_t* map = sm_die_map(&n0, &n1);
    if (map && ntiles >= 2 * clusters) {
      shd.sm_die = map;
      shd.die_split = (int)((ntiles * (n0 / 2) + (n0 / 2 + n1 / 2) / 2) / (n0 / 2 + n1 / 2));
    }
  }
  ProfScope _prof(tag, st);
  kern<<<2 * clusters, tc::kThreads, L::TOTAL, st>>>(a0, a1, b0, b1, shd, epi);
  PPO_LAUNCH_CHECK("tc_gemm2_kernel");
  return PPO_OK;
}

// Two CTA pairs sharing B by multicast (cluster of 4): 512 x 256 per cluster, K-major A and B.
template <class Epi>
int launch2mc(const char* tag, const CUtensorMap& a0, const CUtensorMap& b0,
              const tc::TileShape& sh, const Epi& epi, cudaStream_t st) {
  constexpr int STAGES = 7;   // 7 x 32 KB: the two pairs release a stage only together
  using L = tc::SmemMC<STAGES>;
  auto kern = tc::tc_gemm2mc_kernel<STAGES, Epi>;
  static bool configured = false;
  if (!configured) {
    PPO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL));
    configured = true;
  }
  if (sh.nkb0 <= 0 || sh.nkb1 != 0 || sh.ksplit > 1)
    return fail(PPO_E_SHAPE, "multicast pair kernel: one K source, no split");
  if (!sh.sched) return fail(PPO_E_CUDA, "tile scheduler counter unavailable");
  const int64_t num_m = (sh.M + 255) / 256;
  const int64_t units = ((num_m + 1) / 2) * ((sh.N + 255) / 256);
  const int clusters = (int)std::min<int64_t>(units, num_sms() / 4);
  if (clusters <= 0) return PPO_OK;
  ProfScope _prof(tag, st);
  kern<<<4 * clusters, tc::kThreads, L::TOTAL, st>>>(a0, b0, sh, epi);
  PPO_LAUNCH_CHECK("tc_gemm2mc_kernel");
  return PPO_OK;
}

// Two CTA pairs sharing A by multicast (cluster of 4, MB = 2): 512 x 512 per cluster,
// MN-major A and B (the weight gradient).
template <class Epi>
int launch2mca(const char* tag, const CUtensorMap& a0, const CUtensorMap& b0,
               const tc::TileShape& sh, const Epi& epi, cudaStream_t st) {
  constexpr int STAGES = 4;   // 4 x 48 KB
  using L = tc::SmemMCA<STAGES>;
  auto kern = tc::tc_gemm2mca_kernel<STAGES, Epi>;
  static bool configured = false;
  if (!configured) {
    PPO_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL));
    configured = true;
  }
  if (sh.nkb0 <= 0 || sh.nkb1 != 0 || sh.ksplit > 1 || sh.tsteps > 1)
    return fail(PPO_E_SHAPE, "multicast-A pair kernel: one K source, no split");
  if (!sh.sched) return fail(PPO_E_CUDA, "tile scheduler counter unavailable");
  const int64_t num_n = (sh.N + 255) / 256;
  const int64_t units = ((sh.M + 511) / 512) * ((num_n + 1) / 2);
  int max_clusters = num_sms() / 4;
  {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute attr;
    attr.id = cudaLaunchAttributeClusterDimension;
    attr.val.clusterDim.x = 4;
    attr.val.clusterDim.y = 1;
    attr.val.clusterDim.z = 1;
    cfg.gridDim = dim3(4 * max_clusters);
    cfg.blockDim = dim3(tc::kThreads);
    cfg.dynamicSmemBytes = L::TOTAL;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess && n > 0)
      max_clusters = std::min(max_clusters, n);
    else
      (void)cudaGetLastError();
  }
  const int clusters = (int)std::min<int64_t>(units, max_clusters);
  if (clusters <= 0) return PPO_OK;
  ProfScope _prof(tag, st);
  kern<<<4 * clusters, tc::kThreads, L::TOTAL, st>>>(a0, b0, sh, epi);
  PPO_LAUNCH_CHECK("tc_gemm2mca_kernel");
  return PPO_OK;
}

// The multicast-A kernel's units are pairs of n-tiles: halve an n-grouped raster's group.
tc::TileShape mca_shape(tc::TileShape sh) {
  if (sh.group_n) sh.group = std::max(1, sh.group / 2);
  return sh;
}
inline int cdiv(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

// Split-K factor in [1, kMaxSplitK] that best fills whole waves of `sms` CTAs (each split
// keeps >= 64 k-blocks); 1 when the tiles alone fill the machine.
int pick_split(int tiles, int sms, int nkb) {
  if (tiles >= sms) return 1;
  int best = 1;
  double best_eff = 0.0;
  for (int sp = 1; sp <= kMaxSplitK && nkb / sp >= 64; ++sp) {
    const int units = tiles * sp;
    const int waves = (units + sms - 1) / sms;
    const double eff = (double)units / ((double)waves * sms);
    if (eff > best_eff + 0.02) {
      best_eff = eff;
      best = sp;
    }
  }
  return best;
}

// Raster override for experiments: PPO_RASTER_<KIND>=m<g> or n<g> (e.g. n16).
void raster(tc::TileShape& sh, const char* kind, int def_group, int def_n) {
  sh.group = def_group;
  sh.group_n = def_n;
  char name[64];
  snprintf(name, sizeof(name), "PPO_RASTER_%s", kind);
  const char* e = knob(name);
  if (e && (e[0] == 'm' || e[0] == 'n') && atoi(e + 1) > 0) {
    sh.group_n = e[0] == 'n';
    sh.group = atoi(e + 1);
  }
}

// Kernel variant per GEMM kind (both are tcgen05 paths): CTA pair (256x256, cta_group::2)
// or single CTA (128x256).  Defaults from the energy sweeps (tools/gemm_energy.py; the step
// is power-capped, so TFLOP/J decides); PPO_VARIANT_<KIND>=pair|1cta overrides.
bool use_pair(const char* kind, bool def) {
  char name[64];
  snprintf(name, sizeof(name), "PPO_VARIANT_%s", kind);
  const char* e = knob(name);
  if (!e) return def;
  return strcmp(e, "pair") == 0;
}

struct WsPtrs {
  __nv_bfloat16* xh;
  __nv_bfloat16* g;
  float* c;
  float* dc;
  unsigned int* sched;   // this workspace's tile-scheduler counters, kSchedWords per SchedSlot
  unsigned int* ready;   // multi-step launches: [T][ceil(B / 256)][ready_ld(H)] counters
  size_t counter_bytes;  // sched + ready
  unsigned int* slot(int k) const { return sched + kSchedWords * k; }
};
WsPtrs ws_ptrs(const Shape& s, int64_t B, void* ws) {
  WsLayout L = ws_layout(s, B);
  uint8_t* p = static_cast<uint8_t*>(ws);
  return {reinterpret_cast<__nv_bfloat16*>(p + L.xh), reinterpret_cast<__nv_bfloat16*>(p + L.g),
          reinterpret_cast<float*>(p + L.c), reinterpret_cast<float*>(p + L.dc),
          reinterpret_cast<unsigned int*>(p + L.sched), reinterpret_cast<unsigned int*>(p + L.ready),
          L.ready - L.sched + ready_bytes(s.T, B, s.H)};
}
// zero the workspace's counters on the stream before its GEMMs (fresh memory is arbitrary)
int sched_reset(const WsPtrs& P, cudaStream_t st) {
  ProfScope _prof("sched_reset", st);
  PPO_CUDA_CHECK(cudaMemsetAsync(P.sched, 0, P.counter_bytes, st));
  return PPO_OK;
}
// Fine-grained multi-step dependencies (TileShape::dep_fine): the unit waits for the 64-unit
// blocks it reads, not the whole row block.  Measured slower than the row-block waits (B = 600:
// forward 2.53 vs 2.26 ms, backward as one launch 2.90-3.48 vs 2.44 ms per-step; tiny 575 vs
// 555 us: profiles/r02_fine_deps_ab.txt), so off; PPO_MULTISTEP_FINE=1 (experiment builds).
void fine_deps(tc::TileShape& sh, const Shape& s, bool backward) {
  if (knob_int("PPO_MULTISTEP_FINE", 0) == 0 || s.H % 64 != 0) return;
  if (!backward && s.D % 64 != 0) return;   // h_{t-1} must start on a k-block
  sh.dep_fine = 1;
  sh.dep_ng = (int)(s.H / 64);
  sh.dep_ld = (int)ready_ld(s.H);
  if (backward) {
    // dz_{t+1} columns of unit block j are gate-grouped: 4 k-blocks (one per gate) per block;
    // a 256-unit tile publishes 4 blocks
    sh.dep_kpg = 4;
    sh.epi_q = 4;
    sh.dep_perm = (sh.dep_ng % 4 == 0) && knob_int("PPO_MULTISTEP_PERM", 1) != 0;
  } else {
    // h_{t-1} columns: one k-block per 64 units; a tile (256 gate columns) is one block
    sh.dep_kpg = 1;
    sh.epi_q = 1;
  }
}

// Split-K factor for the backward step GEMM (0 = keep the fused-epilogue launch): only when a
// step has fewer tiles than CTA pairs, on the bf16 path (the partials use the dW_o split-K
// region, which must hold them).  PPO_BWD_SPLIT=0 (experiment builds) keeps the fused path.
int bwd_split(const Shape& s, int64_t B, bool pair, int64_t tiles) {
  if (!pair || !s.bf16 || s.H % 64 != 0 || knob_int("PPO_BWD_SPLIT", 1) == 0) return 0;
  const int clusters = num_sms() / 2;
  if (tiles >= clusters) return 0;
  const int nkb = (int)((s.G4 + s.A_pass + tc::BK - 1) / tc::BK);
  int sp = pick_split((int)tiles, clusters, nkb);
  const size_t room = (size_t)kMaxSplitK * s.A * s.Ko * 4;
  while (sp > 1 && (size_t)sp * B * s.H * 4 > room) --sp;
  // every split of the last step (K = the A_pass head columns only) must get a k-block
  while (sp > 1 && (s.A_pass + tc::BK - 1) / tc::BK < sp) --sp;
  return sp > 1 ? sp : 0;
}

// The T recurrent step GEMMs as ONE persistent launch (tiles of step t+1 start as soon as
// their row block of step t is done, instead of a launch, ramp and tail per step) when a step
// is only a few waves of tiles (small minibatches such as the paper's B = 600); large
// minibatches keep one launch per step (their steps are ~130 waves; nothing to overlap).
// PPO_MULTISTEP=0/1/2 (experiment builds): off / auto / always.
bool use_multistep(int64_t tiles_per_step, bool backward) {
  const int k = knob_int("PPO_MULTISTEP", 1);
  if (k == 0) return false;
  if (k == 2) return true;
  // the backward's A operand is almost all dz_{t+1} (only the 11 dY k-blocks are ready
  // early), so its steps cannot overlap: measured 7% slower than per-step launches at B = 600
  // (profiles/r02_pmb_multistep.txt), but 21% faster in the launch-bound tiny config (one
  // tile per step: r02_tiny_multistep.txt); the forward's x half of K overlaps the previous step
  if (backward) return tiles_per_step <= 4;
  return tiles_per_step <= 8 * (int64_t)(num_sms() / 2);
}

}  // namespace

// Measured once per device, outside stream capture (a capture that needs it runs without);
// NULL when the probe did not find a clean two-die split.
const uint8_t* sm_die_map(int* n0, int* n1) {
  static DieMap maps[64];
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  DieMap& dm = maps[dev];
  if (!dm.done) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(cudaStreamLegacy, &cs);   // (any capture in progress: retry later)
    if (cs != cudaStreamCaptureStatusNone) return nullptr;
    if (probe_die_map(dm) != PPO_OK) dm.dev = nullptr;   // (no map: one queue)
    dm.done = true;
  }
  if (n0) *n0 = dm.n0;
  if (n1) *n1 = dm.n1;
  return dm.dev;
}

// ---------------------------------------------------------------- forward (a2-a4)
int tc_forward(const Shape& s, int64_t B, const void* w, void* ws, float* out,
               const cudaEvent_t* x_ready, cudaStream_t st) {
  WsPtrs P = ws_ptrs(s, B, ws);
  const __nv_bfloat16* wxh = static_cast<const __nv_bfloat16*>(w);
  const __nv_bfloat16* wo = wxh + s.G4 * s.Kx;
  int rc;
  if ((rc = sched_reset(P, st))) return rc;
  // z_t = [x_t | h_{t-1} | 1] W_xh_aug^T : A = XH (3-D, slot t), B = W_xh_aug.
  CUtensorMap mA, mB;
  if ((rc = map_kmajor(&mA, P.xh, s.Kx, B, s.Kx, s.T + 1, B * s.Kx, tc::BM))) return rc;
  const bool pair = use_pair("FWD", true);
  // experiment: PPO_VARIANT_FWD=pair2 -> 512x256 pair tiles (256 A rows per CTA, one
  // 512-column accumulator): 25% less operand traffic per FLOP (the SMs clock ~15% higher
  // under the power cap) but the fused epilogue is no longer overlapped: 15-25% slower
  const char* vf = knob("PPO_VARIANT_FWD");
  const bool pair2 = vf && strcmp(vf, "pair2") == 0;
  // experiment: PPO_VARIANT_FWD=pairmc -> two CTA pairs share the weight tile by 2-SM TMA
  // multicast (cluster of 4): the SMs clock ~10% higher (less L2->SM traffic) but the coupled
  // pairs keep the tensor pipe only ~85% busy (ncu) -> ~8% slower in the step; off
  const bool pairmc = vf && strcmp(vf, "pairmc") == 0;
  CUtensorMap mB1, mA2, mBmc;
  if ((rc = map_kmajor(&mB, wxh, s.Kx, s.G4, s.Kx, 1, 0, 128))) return rc;
  if ((rc = map_kmajor(&mB1, wxh, s.Kx, s.G4, s.Kx, 1, 0, 256))) return rc;
  if (pair2 && (rc = map_kmajor(&mA2, P.xh, s.Kx, B, s.Kx, s.T + 1, B * s.Kx, 256))) return rc;
  if (pairmc && (rc = map_kmajor(&mBmc, wxh, s.Kx, s.G4, s.Kx, 1, 0, 64))) return rc;
  const int64_t fwd_tiles = (int64_t)cdiv(B, 256) * cdiv(s.G4, 256);
  if (pair && !pair2 && !pairmc && !x_ready && s.T > 1 && use_multistep(fwd_tiles, false)) {
    // all T steps in one launch: step t reads XH slot t, its h k-blocks (from column D) wait
    // for step t-1's row block; the epilogue walks XH / C / G by one slot per step
    tc::TileShape sh{(int)B, (int)s.G4, cdiv(s.Kx, tc::BK), 0, 0, 0, 0, 0, 8, 1};
    raster(sh, "FWD", 8, 1);
    sh.sched = P.slot(kSchedFwd);
    sh.tsteps = (int)s.T;
    sh.za_step0 = 1;
    sh.nkb0_s0 = -1;
    sh.dep_kb = (int)(s.D / tc::BK);
    sh.ready = P.ready;
    fine_deps(sh, s, false);
    tc::EpiLstmFwd epi{P.xh + B * s.Kx + s.D, s.Kx, P.c, P.c + B * s.H, P.g, (int)B, (int)s.H,
                       B * s.Kx, B * s.H, B * s.G4};
    CUtensorMap mAi;
    // (the interleaved rows measured 4% slower for the forward's light epilogue:
    // profiles/r02_ilv_tiny.txt; PPO_ILV_FWD=1 in experiment builds)
    if (use_ilv(B) && knob_int("PPO_ILV_FWD", 0) != 0) {
      if ((rc = map_kmajor_ilv(&mAi, P.xh, s.Kx, B, s.Kx, s.T + 1, B * s.Kx))) return rc;
      sh.a_ilv = 1;
      epi.ilv = 1;
    }
    const CUtensorMap& mAx = sh.a_ilv ? mAi : mA;
    if ((rc = launch2<false, false, tc::EpiLstmFwd, 1, 256, true>("lstm_fwd_step", mAx, mAx, mB,
                                                                  mB, sh, epi, st)))
      return rc;
  } else
  for (int t = 0; t < s.T; ++t) {
    if (x_ready && x_ready[t]) PPO_CUDA_CHECK(cudaStreamWaitEvent(st, x_ready[t], 0));
    tc::TileShape sh{(int)B, (int)s.G4, cdiv(s.Kx, tc::BK), 0, t, 0, 0, 0, 8, 1};
    raster(sh, "FWD", 8, 1);
    sh.sched = P.slot(kSchedFwd);
    tc::TileShape sh1 = sh;
    tc::EpiLstmFwd epi{P.xh + (t + 1) * B * s.Kx + s.D, s.Kx, P.c + t * B * s.H,
                       P.c + (t + 1) * B * s.H, P.g + t * B * s.G4, (int)B, (int)s.H, 0, 0, 0};
#ifdef PPO_EXPERIMENTS
    if (pairmc || pair2) {
      rc = pairmc ? launch2mc("lstm_fwd_step", mA, mBmc, sh, epi, st)
                  : launch2<false, false, tc::EpiLstmFwd, 2>("lstm_fwd_step", mA2, mA2, mB, mB,
                                                            sh, epi, st);
      if (rc) return rc;
      continue;
    }
#endif
    rc = pair ? launch2<false, false>("lstm_fwd_step", mA, mA, mB, mB, sh, epi, st)
              : launch<256, false, false>("lstm_fwd_step", mA, mA, mB1, mB1, sh1, epi, st);
    if (rc) return rc;
  }
  // heads: y = [h_t | 1] W_o_aug^T over all T*B rows (XH slots 1..T, columns D..D+Ko).
  // heads: CTA pair, 256 x 224 tiles (3 N-tiles cover A = 656); the 3 N-tiles of a row
  // block run back to back so the head outputs' A rows are read once.
  CUtensorMap hA, hB;
  const bool pair_h = use_pair("HEADS", true);
  if ((rc = map_kmajor(&hA, P.xh + B * s.Kx + s.D, s.Ko, s.T * B, s.Kx, 1, 0, tc::BM))) return rc;
  if ((rc = map_kmajor(&hB, wo, s.Ko, s.A, s.Ko, 1, 0, pair_h ? 112 : 224))) return rc;
  tc::TileShape sh{(int)(s.T * B), (int)s.A, cdiv(s.Ko, tc::BK), 0, 0, 0, 0, 0, 3, 1};
  raster(sh, "HEADS", 3, 1);
  sh.sched = P.slot(kSchedHeads);
  tc::EpiStoreF32 epi{out, s.A, (int)(s.T * B), (int)s.A};
  if (pair_h)
    return launch2<false, false, tc::EpiStoreF32, 1, 224>("heads_fwd", hA, hA, hB, hB, sh, epi, st);
  return launch<224, false, false>("heads_fwd", hA, hA, hB, hB, sh, epi, st);
}

// ---------------------------------------------------------------- backward (a6-a8)
int tc_backward(const Shape& s, int64_t B, const void* w, void* ws, const void* dout, float* grad,
                cudaStream_t st, const DpStage* dp, cudaEvent_t wxh_ready) {
  WsPtrs P = ws_ptrs(s, B, ws);
  const __nv_bfloat16* wxh = static_cast<const __nv_bfloat16*>(w);
  const __nv_bfloat16* wo = wxh + s.G4 * s.Kx;
  const __nv_bfloat16* dY = static_cast<const __nv_bfloat16*>(dout);
  int rc;
  // (the dc carry needs no memset: the t = T-1 epilogue takes it as zero, EpiLstmBwd::first)
  if ((rc = sched_reset(P, st))) return rc;
  // dh_t = dz_{t+1} W_h + dy_t W_o : A = [G (3-D, slot t+1) | dY (3-D, slot t)] (K-major),
  // B = [W_xh_aug[:, D:D+H] | W_o_aug[:, :H]] read MN-major (K = gate row / head output).
  CUtensorMap a0, a1, b0, b1;
  const bool pair = use_pair("BWD", true);
  if ((rc = map_kmajor(&a0, P.g, s.G4, B, s.G4, s.T, B * s.G4, tc::BM))) return rc;
  // only the first A_pass output columns reach the LSTM (stop_gradient aux heads, Q26): the
  // dY / W_o maps end there and TMA zero-fills the rest of the last k-block
  if ((rc = map_kmajor(&a1, dY, s.A_pass, B, s.A, s.T, B * s.A, tc::BM))) return rc;
  if ((rc = map_mnmajor(&b0, wxh + s.D, s.H, s.G4, s.Kx))) return rc;
  if ((rc = map_mnmajor(&b1, wo, s.H, s.A_pass, s.Ko))) return rc;
  const int64_t bwd_tiles = (int64_t)cdiv(B, 256) * cdiv(s.H, 256);
  if (pair && s.T > 1 && use_multistep(bwd_tiles, true)) {
    // all T steps in one launch, step s = time T-1-s: A = [G slot t+1 | dY slot t] (no dz part
    // on step 0), every k-block of the dz part waits for step s-1's row block; the epilogue
    // walks G / C back by one slot per step
    tc::TileShape sh{(int)B, (int)s.H, cdiv(s.G4, tc::BK), cdiv(s.A_pass, tc::BK), (int)s.T,
                     (int)s.T - 1, 0, 0, 8, 1};
    raster(sh, "BWD", 8, 1);
    sh.sched = P.slot(kSchedBwd);
    sh.tsteps = (int)s.T;
    sh.za_step0 = -1;
    sh.za_step1 = -1;
    sh.nkb0_s0 = 0;
    sh.dep_kb = 0;
    sh.ready = P.ready;
    fine_deps(sh, s, true);
    // the dY k-blocks (no dependency) first: they load and multiply while step s-1 finishes
    if (!sh.dep_fine) sh.src1_first = knob_int("PPO_BWD_SRC1_FIRST", 1);
    const int64_t t0 = s.T - 1;
    tc::EpiLstmBwdTail epi{P.g + t0 * B * s.G4, P.c + (t0 + 1) * B * s.H, P.c + t0 * B * s.H,
                           P.dc, (int)B, (int)s.H, 1, knob_int("PPO_EXP_BWD_EPI", 0), -B * s.H,
                           -B * s.G4};
    CUtensorMap a0i, a1i;
    if (use_ilv(B)) {
      if ((rc = map_kmajor_ilv(&a0i, P.g, s.G4, B, s.G4, s.T, B * s.G4))) return rc;
      if ((rc = map_kmajor_ilv(&a1i, dY, s.A_pass, B, s.A, s.T, B * s.A))) return rc;
      sh.a_ilv = 1;
      epi.ilv = 1;
    }
    if ((rc = launch2<false, true, tc::EpiLstmBwdTail, 1, 256, true>(
             "lstm_bwd_step", sh.a_ilv ? a0i : a0, sh.a_ilv ? a1i : a1, b0, b1, sh, epi, st)))
      return rc;
  } else if (const int nsplit = bwd_split(s, B, pair, bwd_tiles)) {
    // small minibatch (fewer tiles per step than CTA pairs, e.g. the paper's B = 600: 48 tiles
    // on 74 pairs, each running the whole K = 4H + A and then an exposed row-per-thread
    // epilogue): split K over nsplit x tiles units (~2 full waves), fp32 partials of dh into
    // the dW_o split-K region, then the cell backward as a coalesced elementwise kernel
    float* part = reinterpret_cast<float*>(static_cast<uint8_t*>(ws) + ws_layout(s, B).splitk);
    for (int t = (int)s.T - 1; t >= 0; --t) {
      const bool last = t == s.T - 1;
      tc::TileShape sh{(int)B, (int)s.H, last ? 0 : cdiv(s.G4, tc::BK), cdiv(s.A_pass, tc::BK),
                       t + 1, t, 0, 0, 8, 1};
      raster(sh, "BWD", 8, 1);
      sh.ksplit = nsplit;
      sh.sched = P.slot(kSchedBwd);
      tc::EpiStoreF32 epi{part, s.H, (int)B, (int)s.H, B * s.H};
      if ((rc = launch2<false, true>("lstm_bwd_step", a0, a1, b0, b1, sh, epi, st))) return rc;
      if ((rc = launch_cell_bwd_split(part, nsplit, B * s.H, P.g + t * B * s.G4,
                                      P.c + (t + 1) * B * s.H, P.c + t * B * s.H, P.dc, B, s.H,
                                      last, st)))
        return rc;
    }
  } else
  for (int t = (int)s.T - 1; t >= 0; --t) {
    const bool last = t == s.T - 1;
    tc::TileShape sh{(int)B, (int)s.H, last ? 0 : cdiv(s.G4, tc::BK), cdiv(s.A_pass, tc::BK),
                     t + 1, t, 0, 0, 8, 1};
    raster(sh, "BWD", 8, 1);   // n8: A/B with the current kernels, backward GEMM 0.7-2 ms faster than n4
    sh.sched = P.slot(kSchedBwd);
    tc::EpiLstmBwd epi{P.g + t * B * s.G4, P.c + (t + 1) * B * s.H, P.c + t * B * s.H, P.dc,
                       (int)B, (int)s.H, last ? 1 : 0,
                       knob_int("PPO_EXP_BWD_EPI", 0), 0, 0};
    tc::TileShape sh1 = sh;
    rc = pair ? launch2<false, true>("lstm_bwd_step", a0, a1, b0, b1, sh, epi, st)
              : launch<256, false, true>("lstm_bwd_step", a0, a1, b0, b1, sh1, epi, st);
    if (rc) return rc;
  }
  // weight gradients: dW_xh_aug = dZ^T [x | h_prev | 1 | 0] over all T*B rows (db falls out
  // of the ones column); dW_o_aug = dY^T [h | 1 | 0].
  CUtensorMap wa, wb, oa, ob;
  const int64_t rows = s.T * B;
  if ((rc = map_mnmajor(&wa, P.g, s.G4, rows, s.G4))) return rc;
  if ((rc = map_mnmajor(&wb, P.xh, s.Kx, rows, s.Kx))) return rc;
  {
    // K = T*B is long (614,400 at the full config): run it as K-chunks of ~153,600 rows, each
    // a separate launch that accumulates into dW.  The tiles of one launch start together and
    // drift apart little over a chunk, so the shared operand panels stay in L2 (DRAM traffic
    // and hence power drop; the step is power-capped).  PPO_WGRAD_CHUNK overrides the rows.
    const int nkb_all = cdiv(rows, tc::BK);
    int chunk_kb = 2400;   // 153,600 rows: A/B on two boxes, dW_xh 4.6% faster than 76,800
    if (const char* e = knob("PPO_WGRAD_CHUNK")) chunk_kb = std::max(1, atoi(e) / tc::BK);
    const int nchunks = std::max(1, (nkb_all + chunk_kb - 1) / chunk_kb);
    const bool pair = use_pair("WGRAD", true);
    // experiment: PPO_VARIANT_WGRAD=pairmc -> two CTA pairs share the dZ panel by multicast
    const char* vw = knob("PPO_VARIANT_WGRAD");
    const bool pairmc = vw && strcmp(vw, "pairmc") == 0;
    for (int c = 0; c < nchunks; ++c) {
      const int kb0 = (int)((int64_t)nkb_all * c / nchunks);
      const int kb1 = (int)((int64_t)nkb_all * (c + 1) / nchunks);
      tc::TileShape sh{(int)s.G4, (int)s.Kx, kb1 - kb0, 0, 0, 0, 0, 0, 8, 0};
      raster(sh, "WGRAD", 8, 1);   // n8: A/B in the step 2-3% faster than m8 (current kernels)
      sh.kb_off = kb0;
      sh.sched = P.slot(kSchedWgrad);
      tc::EpiStoreF32 epi{grad, s.Kx, (int)s.G4, (int)s.Kx, 0, c > 0 ? 1 : 0};
      if (dp && c == nchunks - 1) {
        // the last chunk's tiles are final: their epilogues push them to the DP owners over
        // NVLink while the remaining tiles are still being multiplied
        tc::EpiStoreF32Dp epd{grad, s.Kx, (int)s.G4, (int)s.Kx, 0, c > 0 ? 1 : 0};
        epd.dp = *dp;
#ifdef PPO_EXPERIMENTS
        if (pairmc) rc = launch2mca("wgrad_xh", wa, wb, mca_shape(sh), epd, st);
        else
#endif
        rc = pair ? launch2<true, true, tc::EpiStoreF32Dp, 2>("wgrad_xh", wa, wa, wb, wb, sh, epd,
                                                             st)
                  : launch<256, true, true>("wgrad_xh", wa, wa, wb, wb, sh, epd, st);
      } else {
#ifdef PPO_EXPERIMENTS
        if (pairmc) rc = launch2mca("wgrad_xh", wa, wb, mca_shape(sh), epi, st);
        else
#endif
        rc = pair ? launch2<true, true, tc::EpiStoreF32, 2>("wgrad_xh", wa, wa, wb, wb, sh, epi, st)
                  : launch<256, true, true>("wgrad_xh", wa, wa, wb, wb, sh, epi, st);
      }
      if (rc) return rc;
    }
  }
  // dW_xh (97% of theta) is final here: let the caller start exchanging it (overlapping dW_o)
  if (wxh_ready) PPO_CUDA_CHECK(cudaEventRecord(wxh_ready, st));
  if ((rc = map_mnmajor(&oa, dY, s.A, rows, s.A))) return rc;
  if ((rc = map_mnmajor(&ob, P.xh + B * s.Kx + s.D, s.Ko, rows, s.Kx))) return rc;
  {
    // dW_o has only ceil(A/128) x ceil(Ko/256) = 102 tiles at full size (< 148 SMs) and
    // K = T*B: split K so the grid fills the SMs; partials are reduced in a fixed order.
    tc::TileShape sh{(int)s.A, (int)s.Ko, cdiv(rows, tc::BK), 0, 0, 0, 0, 0, 16, 0};
    const bool pair_o = use_pair("WGRAD_O", true);
    const int tiles = pair_o ? cdiv(s.A, 256) * cdiv(s.Ko, 256) : cdiv(s.A, tc::BM) * cdiv(s.Ko, 256);
    sh.ksplit = pick_split(tiles, pair_o ? num_sms() / 2 : num_sms(), cdiv(rows, tc::BK));
    sh.sched = P.slot(kSchedWgradO);
    float* dwo = grad + s.G4 * s.Kx;
    const int64_t n_o = s.A * s.Ko;
    float* part = sh.ksplit > 1 ? reinterpret_cast<float*>(static_cast<uint8_t*>(ws) +
                                                              ws_layout(s, B).splitk)
                                : dwo;
    tc::EpiStoreF32 epi{part, s.Ko, (int)s.A, (int)s.Ko, n_o};
    if (dp && sh.ksplit == 1) {
      tc::EpiStoreF32Dp epd{part, s.Ko, (int)s.A, (int)s.Ko, n_o};
      epd.dp = *dp;
      epd.dp_base = s.G4 * s.Kx;
      rc = pair_o ? launch2<true, true>("wgrad_o", oa, oa, ob, ob, sh, epd, st)
                  : launch<256, true, true>("wgrad_o", oa, oa, ob, ob, sh, epd, st);
    } else {
      rc = pair_o ? launch2<true, true>("wgrad_o", oa, oa, ob, ob, sh, epi, st)
                  : launch<256, true, true>("wgrad_o", oa, oa, ob, ob, sh, epi, st);
    }
    if (rc) return rc;
    if (sh.ksplit > 1 &&
        (rc = launch_splitk_reduce(part, sh.ksplit, (size_t)n_o, dwo, st, dp, s.G4 * s.Kx)))
      return rc;
    if (s.win_pass &&  // dout's win column carries win_trunk x the gradient (Q26)
        (rc = launch_scale(dwo + (int64_t)(s.vcol + 1) * s.Ko, s.Ko, 1.f / s.win_trunk, st)))
      return rc;
  }
  return PPO_OK;
}

// ---------------------------------------------------------------- NEXT-4: dL/dx
// dX[t][b] = dz_t[b] W_x for all t at once: A = dz (G, [T*B][4H] K-major), B = W_x (the
// first D columns of W_xh_aug, MN-major [4H][D] with ld Kx); CTA-pair 256x256 tiles.
int tc_input_grad(const Shape& s, int64_t B, const void* w, void* ws, float* dx, cudaStream_t st) {
  WsPtrs P = ws_ptrs(s, B, ws);
  const __nv_bfloat16* wxh = static_cast<const __nv_bfloat16*>(w);
  const int64_t rows = s.T * B;
  CUtensorMap ma, mb;
  int rc;
  if ((rc = map_kmajor(&ma, P.g, s.G4, rows, s.G4, 1, 0, tc::BM))) return rc;
  if ((rc = map_mnmajor(&mb, wxh, s.D, s.G4, s.Kx))) return rc;
  if ((rc = sched_reset(P, st))) return rc;
  tc::TileShape sh{(int)rows, (int)s.D, cdiv(s.G4, tc::BK), 0, 0, 0, 0, 0, 8, 0};
  raster(sh, "DX", 8, 0);
  sh.sched = P.slot(kSchedDx);
  tc::EpiStoreF32 epi{dx, s.D, (int)rows, (int)s.D};
  return launch2<false, true>("input_grad", ma, ma, mb, mb, sh, epi, st);
}

// ---------------------------------------------------------------- NEXT-3 inference GEMMs
// Skinny GEMMs of one policy step at batch B ~ 60: the weights are the M side
// (128-row tiles streamed once by TMA, 8-stage ring), the batch the N side (one 64-wide
// tile), K split so the units fill whole waves of the SMs.  Deterministic fp32 partials
// out[split][b][m] (transposed store); the consumer kernel sums them in split order.
namespace {
int infer_split(int tiles, int nkb, int min_kb, const char* knob = "PPO_INFER_SPLIT") {
  const char* e = ppo::knob(knob);
  if (e && atoi(e) > 0) return std::min(std::min(atoi(e), kMaxSplitK), nkb);
  const int sms = num_sms();
  if (tiles >= sms) return 1;   // the tiles alone fill the machine
  int best = 1;
  double best_eff = 0.0;
  // best wave fill; among (near-)ties the larger split (more CTAs streaming the weights).
  // Each split keeps >= min_kb k-blocks, which bounds the fp32 partials the consumer reads.
  for (int sp = 1; sp <= kMaxSplitK && nkb / sp >= min_kb; ++sp) {
    const int units = tiles * sp;
    const double eff = (double)units / ((double)((units + sms - 1) / sms) * sms);
    if (eff > best_eff + 0.02) best_eff = eff;
    if (eff >= best_eff - 0.02) best = sp;
  }
  return best;
}

// N tile by batch size: 64 at the paper's ~60, wider tiles once the batch fills them (the
// MMA needs N >= 128 to stop being shared-memory bound).
// W is pre-tiled (tc_infer_tile_weights): [ceil(M/128) * nkb] tiles of [128][64] bf16.
// The batch operand is the K-concatenation of act0 [B][K0] (ld0) and act1 [B][K - K0] (ld1)
// (K0 = K: one source); K0 must be a multiple of 64.
template <int BN>
int infer_gemm_bn(const char* tag, int slot, const void* W, int64_t M, int64_t K,
                  const void* act0, int64_t K0, int64_t ld0, const void* act1, int64_t ld1,
                  int64_t B, float* part, int* split_out, unsigned int* sched, cudaStream_t st) {
  CUtensorMap ma, mb0, mb1;
  int rc;
  const int nkb = cdiv(K, tc::BK);
  const int64_t wtiles = (int64_t)cdiv(M, tc::BM) * nkb;
  if ((rc = make_map(&ma, W, tc::BK, tc::BM, wtiles, tc::BK * 2, tc::BK * tc::BM * 2, tc::BK,
                     tc::BM)))
    return rc;
  if (K0 % tc::BK) return fail(PPO_E_SHAPE, "first K source must be a multiple of 64");
  if ((rc = map_kmajor(&mb0, act0, K0, B, ld0, 1, 0, BN))) return rc;
  if (K0 < K && (rc = map_kmajor(&mb1, act1, K - K0, B, ld1, 1, 0, BN))) return rc;
  if (K0 == K) mb1 = mb0;
  const int nkb0 = (int)(K0 / tc::BK);
  const int tiles = cdiv(M, tc::BM) * cdiv(B, BN);
  // gates: >= 32 k-blocks per split (4 splits of W_xh at the paper's size: the cell kernel
  // reads 4 partials); heads: >= 8 (8 splits of the small W_o)
  const bool heads = slot == kSchedInferHeads;
  const int sp = infer_split(tiles, nkb, heads ? 8 : 32,
                             heads ? "PPO_INFER_SPLIT_HEADS" : "PPO_INFER_SPLIT");
  tc::TileShape sh{(int)M, (int)B, nkb0, nkb - nkb0, 0, 0, 0, 0, 1, 0};
  sh.ksplit = sp;
  sh.sched = sched + kSchedWords * slot;
  const char* e = knob("PPO_INFER_EVICT_FIRST");
  sh.a_evict_first = e ? atoi(e) : 1;
  sh.a_tiled_nkb = nkb;
  tc::EpiStoreF32T epi{part, M, (int)M, (int)B, M * B};
  *split_out = sp;
  constexpr int STAGES = BN == 64 ? 8 : BN == 128 ? 6 : 4;
  return launch<BN, false, false, tc::EpiStoreF32T, STAGES>(tag, ma, ma, mb0, mb1, sh, epi, st,
                                                             true);
}
int infer_gemm(const char* tag, int slot, const void* W, int64_t M, int64_t K, const void* act0,
               int64_t K0, int64_t ld0, const void* act1, int64_t ld1, int64_t B, float* part,
               int* split_out, unsigned int* sched, cudaStream_t st) {
  if (B <= 64)
    return infer_gemm_bn<64>(tag, slot, W, M, K, act0, K0, ld0, act1, ld1, B, part, split_out,
                             sched, st);
  if (B <= 128)
    return infer_gemm_bn<128>(tag, slot, W, M, K, act0, K0, ld0, act1, ld1, B, part, split_out,
                              sched, st);
  return infer_gemm_bn<256>(tag, slot, W, M, K, act0, K0, ld0, act1, ld1, B, part, split_out,
                            sched, st);
}

}  // namespace

size_t tc_infer_tiled_offset_heads(const Shape& s) {
  return (size_t)cdiv(s.G4, tc::BM) * cdiv(s.Kx, tc::BK) * tc::BM * tc::BK;  // elements
}
size_t tc_infer_tiled_elems(const Shape& s) {
  return tc_infer_tiled_offset_heads(s) + (size_t)cdiv(s.A, tc::BM) * cdiv(s.Ko, tc::BK) * tc::BM * tc::BK;
}
int tc_infer_gates(const Shape& s, int64_t B, const void* wt, const void* x, const void* ho,
                   float* part, int* split, unsigned int* sched, cudaStream_t st) {
  // [x | h | 1 | 0] = x [B][D] straight from the caller, then the state buffer HO [B][Ko]
  return infer_gemm("infer_gates", kSchedInferGates, wt, s.G4, s.Kx, x, s.D, s.D, ho, s.Ko, B,
                    part, split, sched, st);
}
int tc_infer_heads(const Shape& s, int64_t B, const void* wt, const void* ho, float* part,
                   int* split, unsigned int* sched, cudaStream_t st) {
  const __nv_bfloat16* wo = static_cast<const __nv_bfloat16*>(wt) + tc_infer_tiled_offset_heads(s);
  return infer_gemm("infer_heads", kSchedInferHeads, wo, s.A, s.Ko, ho, s.Ko, s.Ko, nullptr, 0, B,
                    part, split, sched, st);
}
int tc_infer_max_split() { return kMaxSplitK; }

// ---------------------------------------------------------------- standalone test GEMM
// mode bit0: B is MN-major ([K][N]) else K-major ([N][K]); bit1: A is MN-major ([K][M]).
// mode bit2: BN = 224 (only with K-major A and B).  C [M][N] fp32.
int tc_test_gemm(int mode, const void* A, const void* Bm, float* C, int M, int N, int K,
                 cudaStream_t st) {
  const bool b_mn = mode & 1, a_mn = mode & 2, n224 = mode & 4, pair = mode & 8;
  CUtensorMap ma, mb;
  int rc;
  const int BN = n224 ? 224 : 256;
  if (a_mn) rc = map_mnmajor(&ma, A, M, K, M);
  else rc = map_kmajor(&ma, A, K, M, K, 1, 0, tc::BM);
  if (rc) return rc;
  if (b_mn) rc = map_mnmajor(&mb, Bm, N, K, N);
  else rc = map_kmajor(&mb, Bm, K, N, K, 1, 0, pair ? 128 : BN);
  if (rc) return rc;
  tc::TileShape sh{M, N, cdiv(K, tc::BK), 0, 0, 0, 0, 0, 16, 0};
  raster(sh, "TEST", 16, 0);
  sh.sched = test_sched_counter();
  tc::EpiStoreF32 epi{C, N, M, N};
  const bool wide = mode & 16, n224p = mode & 32;
  if (pair && n224p) {
    if (a_mn || b_mn) return fail(PPO_E_ARG, "pair N=224 test only for K-major operands");
    CUtensorMap mb2;
    if ((rc = map_kmajor(&mb2, Bm, K, N, K, 1, 0, 112))) return rc;
    return launch2<false, false, tc::EpiStoreF32, 1, 224>("test_gemm2n224", ma, ma, mb2, mb2, sh,
                                                           epi, st);
  }
  if (pair && wide) {
    if (a_mn && b_mn)
      return launch2<true, true, tc::EpiStoreF32, 2>("test_gemm2w", ma, ma, mb, mb, sh, epi, st);
    return fail(PPO_E_ARG, "512-row pair tiles: test mode only for MN-major A and B");
  }
  if (pair) {
    if (!a_mn && !b_mn) return launch2<false, false>("test_gemm2", ma, ma, mb, mb, sh, epi, st);
    if (!a_mn && b_mn) return launch2<false, true>("test_gemm2", ma, ma, mb, mb, sh, epi, st);
    if (a_mn && b_mn) return launch2<true, true>("test_gemm2", ma, ma, mb, mb, sh, epi, st);
    return fail(PPO_E_ARG, "unsupported test mode");
  }
  if (n224) {
    if (a_mn || b_mn) return fail(PPO_E_ARG, "BN=224 test only for K-major operands");
    return launch<224, false, false>("test_gemm", ma, ma, mb, mb, sh, epi, st);
  }
  if (!a_mn && !b_mn) return launch<256, false, false>("test_gemm", ma, ma, mb, mb, sh, epi, st);
  if (!a_mn && b_mn) return launch<256, false, true>("test_gemm", ma, ma, mb, mb, sh, epi, st);
  if (a_mn && b_mn) return launch<256, true, true>("test_gemm", ma, ma, mb, mb, sh, epi, st);
  return fail(PPO_E_ARG, "unsupported test mode");
}

}  // namespace ppo

extern "C" int ppo_device_info(int32_t* n_sms, int32_t* die0_sms, int32_t* die1_sms) {
  if (!n_sms || !die0_sms || !die1_sms) return ppo::fail(PPO_E_ARG, "NULL pointer");
  int n0 = 0, n1 = 0;
  const uint8_t* m = ppo::sm_die_map(&n0, &n1);
  *n_sms = ppo::num_sms();
  *die0_sms = m ? n0 : 0;
  *die1_sms = m ? n1 : 0;
  return PPO_OK;
}

#ifdef PPO_TRACE
// experiments build only: the phase trace of the last pair-GEMM launch (tc_gemm.cuh)
extern "C" int ppo_trace_read(unsigned long long* out, int n) {
  n = std::min(n, 512 * 32);
  return cudaMemcpyFromSymbol(out, ppo::tc::g_tc_trace, n * sizeof(unsigned long long)) ==
                 cudaSuccess
             ? PPO_OK
             : PPO_E_CUDA;
}
extern "C" int ppo_trace_clear(void) {
  static unsigned long long z[512 * 32] = {};
  return cudaMemcpyToSymbol(ppo::tc::g_tc_trace, z, sizeof(z)) == cudaSuccess ? PPO_OK : PPO_E_CUDA;
}
#endif
