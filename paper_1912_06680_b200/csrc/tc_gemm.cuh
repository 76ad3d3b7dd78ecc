// tc_gemm.cuh -- persistent warp-specialised tcgen05 GEMM for sm_100a.
//
//   C[m][n] = sum_k A(m,k) B(n,k),  bf16 operands, fp32 accumulator in TMEM.
//
// Roles (192 threads, 1 CTA/SM):
//   warp 0 lane 0 : TMA producer   (cp.async.bulk.tensor, 128B swizzle, mbarrier ring)
//   warp 1        : TMEM allocator; lane 0 issues tcgen05.mma (M=128, N=BN, K=16)
//   warps 2..5    : epilogue (tcgen05.ld -> registers -> fused functor -> global)
// Two TMEM accumulators (2 x BN columns) so the epilogue of tile i overlaps the
// mainloop of tile i+1.  A and B may each be the K-concatenation of two sources
// (separate tensor maps), split at k-block nkb0; each operand is K-major or MN-major.
#pragma once
#include "common.cuh"

namespace ppo {
namespace tc {

constexpr int BM = 128;
constexpr int BK = 64;             // one 128-byte swizzle row of bf16
constexpr int kThreads = 192;
#ifndef PPO_SUSPEND_HINT_NS
#define PPO_SUSPEND_HINT_NS 1000000
#endif
constexpr uint32_t kSuspendHintNs = PPO_SUSPEND_HINT_NS;

struct TileShape {
  int M, N;          // logical output extent (tiles beyond are masked by the epilogue)
  int nkb0, nkb1;    // k-blocks taken from source 0 / source 1
  int za0, za1;      // 3rd TMA coordinate (time slot) for A sources
  int zb0, zb1;      // ... for B sources
  int group;         // rasterisation: tiles per group along the grouped dimension
  int group_n;       // 0: groups of `group` m-tiles sweep all n; 1: groups of n-tiles sweep m
  int ksplit;        // single-CTA kernel: split K into this many ranges (<= 1: no split); the
                     // epilogue receives the split index and writes a partial result
  int kb_off;        // k-block offset added to source-0 K coordinates (K-chunked launches)
  unsigned int* sched;  // dynamic tile scheduler: {next unit, exited fetchers}, zero at launch;
                        // the last fetcher resets both (one launch per counter at a time)
  int a_evict_first;    // single-CTA kernel, K-major A: L2 evict_first hint on A's TMA loads
                        // (an operand streamed once, e.g. the weights of the inference GEMMs)
  int a_tiled_nkb;      // > 0: A is pre-tiled (16 KB [128 rows][64 k] tiles, tile index
                        // m_tile * a_tiled_nkb + k_block, map dims {64, 128, tiles}) so every
                        // TMA box is one contiguous DRAM stream
  const uint8_t* sm_die;  // CTA-pair kernel: SM -> die map (nullable = one queue)
  int die_split;          // > 0: units [0, die_split) are die 0's queue (sched_fetch_die)
  // CTA-pair kernel, persistent multi-step launch (tsteps > 1): the T recurrent steps of the
  // LSTM in one launch, units = tsteps x tiles in step order (unit step s is passed to the
  // epilogue as `split`).  Step s reads the A sources at 3rd coordinate za{0,1} + s za_step{0,1},
  // takes nkb0_s0 (>= 0) source-0 k-blocks on step 0, and its k-blocks from dep_kb on wait
  // until every tile of step s-1 in the same row block has signalled ready[(s-1) num_m + mb]
  // (2 per tile: both CTAs of the pair, after their epilogue's stores).
  int tsteps;
  int za_step0, za_step1;
  int nkb0_s0;
  int dep_kb;
  unsigned int* ready;
  // Fine-grained dependencies (dep_fine = 1): instead of a whole row block, a unit waits only
  // for the 64-unit blocks of the previous step it reads.  Counters ready[(s num_m + mb) dep_ld
  // + j] count the CTAs (2 per pair) that stored hidden-unit block j of row block mb at step s;
  // k-block kb >= dep_kb of step s reads block j = (kb - dep_kb) / dep_kpg (if j < dep_ng), and
  // a tile's epilogue publishes its epi_q blocks one by one.
  int dep_fine;
  int dep_kpg, dep_ng, dep_ld, epi_q;
  int dep_perm;
  int src1_first;   // multi-step: take source 1's k-blocks before source 0's
  // multi-step, one 256-row tile: the A maps are 4-D row-interleaved views {k, i, q, z} of
  // [rows][k] (row = 4 i + q), so TMEM lane 32 q + i of a CTA holds its row 4 i + q and the
  // valid rows of a small batch spread over all four epilogue warps (Epi::ilv maps back)
  int a_ilv;
};

// One work unit of a launch: a tile and (split-K) its k-range or (multi-step) its step.
struct UnitInfo {
  int split, tile, kb_lo, kb_hi, nkb0, za0, za1;
};
template <bool MS = false>
__device__ __forceinline__ UnitInfo decode_unit(const TileShape& sh, int u, int ntiles) {
  UnitInfo r;
  r.split = u / ntiles;
  r.tile = u - r.split * ntiles;
  if (MS && sh.tsteps > 1) {
    r.nkb0 = (r.split == 0 && sh.nkb0_s0 >= 0) ? sh.nkb0_s0 : sh.nkb0;
    r.kb_lo = 0;
    r.kb_hi = r.nkb0 + sh.nkb1;
    r.za0 = sh.za0 + r.split * sh.za_step0;
    r.za1 = sh.za1 + r.split * sh.za_step1;
  } else {
    const int nsplit = sh.ksplit > 1 ? sh.ksplit : 1, nkb = sh.nkb0 + sh.nkb1;
    r.nkb0 = sh.nkb0;
    r.kb_lo = r.split * nkb / nsplit;
    r.kb_hi = (r.split + 1) * nkb / nsplit;
    r.za0 = sh.za0;
    r.za1 = sh.za1;
  }
  return r;
}
// Multi-step dependencies: spin (acquire, with back-off) until *p >= target.  async = the
// caller then reads the data by TMA (async proxy): order those reads after the acquire.
__device__ __forceinline__ void wait_ready(const unsigned int* p, unsigned int target,
                                           bool async) {
  unsigned int v;
  uint32_t spins = 0;
  while (true) {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if (v >= target) break;
    __nanosleep(128);
    if (++spins == (1u << 26)) asm volatile("trap;");   // watchdog (~10 s)
  }
  if (async) asm volatile("fence.proxy.async.global;" ::: "memory");
}
// Fine-grained dependencies: poll the 8 counters of group j's aligned octet (two acquire 16-byte
// loads) until counter j reaches target; returns the octet's ready bits (bit i: counter
// (j & ~7) + i) so the caller skips the polls of groups already seen ready (a full fence here
// instead of acquire loads stalls the producer behind its own TMA loads); async = then order
// TMA reads after it.
__device__ __forceinline__ uint32_t wait_group(const unsigned int* row, int j, unsigned int target,
                                               bool async) {
  const unsigned int* p = row + (j & ~7);
  uint32_t bits = 0;
  uint32_t spins = 0;
  while (true) {
    unsigned int v[8];
    asm volatile("ld.acquire.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "l"(p) : "memory");
    asm volatile("ld.acquire.gpu.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]) : "l"(p + 4) : "memory");
    bits = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) bits |= (v[i] >= target ? 1u : 0u) << i;
    if ((bits >> (j & 7)) & 1u) break;
    __nanosleep(64);
    if (++spins == (1u << 26)) asm volatile("trap;");   // watchdog
  }
  if (async) asm volatile("fence.proxy.async.global;" ::: "memory");
  return bits;
}
constexpr int kSchedDepth = 4;  // tile-index ring between the fetcher and the consumers
// Blocks of 64 hidden units a 256-column tile of an LSTM epilogue publishes under fine-grained
// multi-step dependencies (Epi::kFineBlocks; 0 = not an LSTM step epilogue)
template <class E, class = void>
struct FineBlocks {
  static constexpr int v = 0;
};
template <class E>
struct FineBlocks<E, std::void_t<decltype(E::kFineBlocks)>> {
  static constexpr int v = E::kFineBlocks;
};

// ---------------------------------------------------------------- PTX wrappers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Wait for the phase with the given parity.  try_wait carries a suspend-time hint so a
// waiting warp sleeps in hardware instead of re-issuing polls (energy: the step is
// power-capped).  Watchdog: a wait longer than 20 s traps (a pipeline bug then surfaces as a
// launch error instead of a hung GPU).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  uint32_t done;
  uint32_t spins = 0;
  uint64_t t0 = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity), "r"(kSuspendHintNs)
        : "memory");
    if (!done && ((++spins & 0xFFu) == 0)) {
      const uint64_t now = globaltimer_ns();
      if (t0 == 0) t0 = now;
      else if (now - t0 > 20000000000ull) asm volatile("trap;");
    }
  } while (!done);
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_3d_hint(const CUtensorMap* map, uint64_t* bar, void* dst,
                                                 int c0, int c1, int c2, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
// SMEM matrix descriptor (tcgen05 "shared memory descriptor"): start>>4 [0,14),
// LBO>>4 [16,30), SBO>>4 [32,46), version=1 [46,48), base offset 0, layout
// SWIZZLE_128B (=2) in [61,64).
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(2) << 61;
  return d;
}
// Instruction descriptor, kind::f16: D=f32 [4,6), A=bf16 [7,10), B=bf16 [10,13),
// a_major [15], b_major [16] (1 = MN-major), N>>3 [17,23), M>>4 [24,29).
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) |
         ((b_mn ? 1u : 0u) << 16) | (static_cast<uint32_t>(N >> 3) << 17) |
         (static_cast<uint32_t>(M >> 4) << 24);
}
__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t ad, uint64_t bd,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}
// 32 lanes x 16 consecutive fp32 columns; waits for completion before returning.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  __syncwarp();  // .sync.aligned: the whole warp executes this convergently
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}


// One lane of a converged warp (the lowest active one: always the same lane, so tcgen05.commit
// tracks the MMAs that lane issued).
__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred P;\n\t"
      "elect.sync _|P, 0xffffffff;\n\t"
      "selp.b32 %0, 1, 0, P;\n\t}"
      : "+r"(pred));
  return pred != 0;
}

// ---- CTA-pair (cta_group::2) helpers ----------------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA into this CTA's smem, completion counted on the leader CTA's mbarrier (cluster address).
__device__ __forceinline__ void tma_load_3d_pair(const CUtensorMap* map, uint32_t bar_cluster,
                                                 void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
__device__ __forceinline__ void tma_load_4d_pair(const CUtensorMap* map, uint32_t bar_cluster,
                                                 void* dst, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t ad, uint64_t bd,
                                               uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(ad), "l"(bd), "r"(idesc), "r"(accumulate)
      : "memory");
}
// Arrive (when all prior MMAs of this thread complete) on the barrier at the same smem
// offset in both CTAs of the pair.
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster)
               : "memory");
}
__device__ __forceinline__ void st_shared_cluster(uint32_t addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// Wait on a local barrier that a peer CTA arrives on (acquire at cluster scope).
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  uint32_t done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity), "r"(kSuspendHintNs)
        : "memory");
  } while (!done);
}
// Fetch the next work unit from the global counter; the fetcher that observes the end last
// resets the counter for the next launch.  ctr[0] = next unit, ctr[1] = exited fetchers.
__device__ __forceinline__ int sched_fetch(unsigned int* ctr, int nunits, unsigned int nfetchers) {
  const int u = static_cast<int>(atomicAdd(ctr, 1u));
  if (u >= nunits && atomicAdd(ctr + 1, 1u) == nfetchers - 1) {
    atomicExch(ctr, 0u);
    atomicExch(ctr + 1, 0u);
  }
  return u;
}
// Die-aware variant (split > 0): units [0, split) are die 0's queue (ctr[0]), [split, nunits)
// die 1's (ctr[2]); each fetcher takes from its own die's queue in raster order, so the tiles
// that share operand panels run on one die and the panels are fetched into that die's L2
// (fewer cross-die fabric transfers); an exhausted queue steals from the other one.
__device__ __forceinline__ int sched_fetch_die(unsigned int* ctr, int nunits,
                                               unsigned int nfetchers, int die, int split) {
#pragma unroll
  for (int k = 0; k < 2; ++k) {
    const int d = die ^ k;
    const int u = static_cast<int>(atomicAdd(ctr + 2 * d, 1u));
    if (u < (d ? nunits - split : split)) return (d ? split : 0) + u;
  }
  if (atomicAdd(ctr + 1, 1u) == nfetchers - 1) {
    atomicExch(ctr, 0u);
    atomicExch(ctr + 1, 0u);
    atomicExch(ctr + 2, 0u);
  }
  return nunits;
}
__device__ __forceinline__ uint32_t smid() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
  return r;
}

// ---------------------------------------------------------------- phase trace (experiments)
// Built with -DPPO_TRACE only: per CTA, clock64() at phase points relative to kernel entry
// (slot 0 holds %globaltimer at entry), read back by ppo_trace_read (tools/trace_gemm.py).
#ifdef PPO_TRACE
__device__ unsigned long long g_tc_trace[512][32];
__device__ __forceinline__ void tc_trace(int i, long long t0) {
  g_tc_trace[blockIdx.x][i] = (unsigned long long)(clock64() - t0);
}
#define TC_TRACE(i) tc_trace((i), trace_t0)
#ifdef PPO_TRACE_UNIT   // trace the unit with this index (multi-step: step s of tile 0 = s)
#define TC_SEL(u, first) ((u) == PPO_TRACE_UNIT)
#else                   // trace the CTA's first unit
#define TC_SEL(u, first) (first)
#endif
#define TC_TRACE_BEGIN()                                                 \
  const long long trace_t0 = clock64();                                  \
  if (threadIdx.x == 0) g_tc_trace[blockIdx.x][0] = globaltimer_ns()
#else
#define TC_TRACE(i) \
  do {              \
  } while (0)
#define TC_SEL(u, first) false
#define TC_TRACE_BEGIN() \
  do {                   \
  } while (0)
#endif

// ---------------------------------------------------------------- the kernel
template <int BN, bool A_MN, bool B_MN, int STAGES>
struct Smem {
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + (2 * STAGES + 4 + 2 * kSchedDepth) * 8 + 32 + 1024;
};

// Grouped rasterisation: consecutive tiles (which run concurrently) share a group of
// `group` m-tiles (group_n = 0) or n-tiles (group_n = 1) and sweep the other dimension, so
// the group's operand panels stay in L2 while the other operand streams through once.
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int group,
                                            int group_n, int& mb, int& nb) {
  if (group_n) {
    const int per_group = group * num_m;
    const int g = tile / per_group;
    const int first_n = g * group;
    const int gsz = min(group, num_n - first_n);
    const int local = tile - g * per_group;
    nb = first_n + local % gsz;
    mb = local / gsz;
  } else {
    const int per_group = group * num_n;
    const int g = tile / per_group;
    const int first_m = g * group;
    const int gsz = min(group, num_m - first_m);
    const int local = tile - g * per_group;
    mb = first_m + local % gsz;
    nb = local / gsz;
  }
}

template <int BN, bool A_MN, bool B_MN, int STAGES, class Epi>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap ta1,
                   const __grid_constant__ CUtensorMap tb0, const __grid_constant__ CUtensorMap tb1,
                   const TileShape sh, const Epi epi) {
  using L = Smem<BN, A_MN, B_MN, STAGES>;
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N");
  static_assert(!B_MN || BN % 64 == 0, "MN-major B needs 64-wide panels");
  extern __shared__ uint8_t smem_raw[];
  // 128B-swizzled TMA/UMMA tiles need 1024-byte aligned shared addresses
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;              // tile-index ring: filled
  uint64_t* sempty = sfull + kSchedDepth;    //                  consumed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sempty + kSchedDepth);
  int* ring = reinterpret_cast<int*>(tslot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int num_m = (sh.M + BM - 1) / BM;
  const int num_n = (sh.N + BN - 1) / BN;
  const int ntiles = num_m * num_n;
  const int nkb = sh.nkb0 + sh.nkb1;
  const int nsplit = sh.ksplit > 1 ? sh.ksplit : 1;
  const int nunits = ntiles * nsplit;

  if (threadIdx.x == 0) {
    prefetch_map(&ta0);
    prefetch_map(&tb0);
    if (sh.nkb1 > 0) {
      prefetch_map(&ta1);
      prefetch_map(&tb1);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    for (int s = 0; s < kSchedDepth; ++s) {
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 5);  // MMA warp + 4 epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // Programmatic dependent launch (no-ops without the launch attribute): the set-up above
  // overlaps the previous kernel's tail; operands are read only after it has completed.
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      // ===================== TMA producer =====================
      // also the tile-scheduler fetcher: units are handed out in order from a global
      // counter, so the tiles in flight stay contiguous in raster order (L2 locality)
      int stage = 0;
      uint32_t phase = 0;
      int sslot = 0;
      uint32_t sphase = 0;
      while (true) {
        mbar_wait(&sempty[sslot], sphase ^ 1);
        const int unit = sched_fetch(sh.sched, nunits, gridDim.x);
        ring[sslot] = unit;
        mbar_arrive(&sfull[sslot]);
        if (++sslot == kSchedDepth) {
          sslot = 0;
          sphase ^= 1;
        }
        if (unit >= nunits) break;
        const int split = unit / ntiles, tile = unit - split * ntiles;
        int mb, nb;
        tile_coords(tile, num_m, num_n, sh.group, sh.group_n, mb, nb);
        const int kb_lo = split * nkb / nsplit, kb_hi = (split + 1) * nkb / nsplit;
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], L::STAGE_BYTES);
          const bool s1 = kb >= sh.nkb0;
          const int kk = (s1 ? kb - sh.nkb0 : kb + sh.kb_off) * BK;
          const CUtensorMap* ta = s1 ? &ta1 : &ta0;
          const CUtensorMap* tb = s1 ? &tb1 : &tb0;
          const int za = s1 ? sh.za1 : sh.za0;
          const int zb = s1 ? sh.zb1 : sh.zb0;
          uint8_t* a_dst = sA + stage * L::A_BYTES;
          uint8_t* b_dst = sB + stage * L::B_BYTES;
          if (!A_MN) {
            const int a0 = sh.a_tiled_nkb ? 0 : kk;
            const int a1 = sh.a_tiled_nkb ? 0 : mb * BM;
            const int a2 = sh.a_tiled_nkb ? mb * sh.a_tiled_nkb + kb : za;   // global k-block
            if (sh.a_evict_first)
              tma_load_3d_hint(ta, &full[stage], a_dst, a0, a1, a2, policy_evict_first());
            else
              tma_load_3d(ta, &full[stage], a_dst, a0, a1, a2);
          } else {
#pragma unroll
            for (int p = 0; p < BM / 64; ++p)
              tma_load_3d(ta, &full[stage], a_dst + p * (BK * 128), mb * BM + p * 64, kk, za);
          }
          if (!B_MN) {
            tma_load_3d(tb, &full[stage], b_dst, kk, nb * BN, zb);
          } else {
#pragma unroll
            for (int p = 0; p < BN / 64; ++p)
              tma_load_3d(tb, &full[stage], b_dst + p * (BK * 128), nb * BN + p * 64, kk, zb);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer: the warp waits, one elected lane issues ===========
    // Descriptors are built once for stage 0 and advanced by adding to the 14-bit start
    // address field (stage: bytes>>4; UMMA_K step: 32 B K-major, 16 rows x 128 B MN-major).
    constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
    const uint64_t a_desc0 = A_MN ? sdesc(smem_u32(sA), BK * 128, 1024) : sdesc(smem_u32(sA), 16, 1024);
    const uint64_t b_desc0 = B_MN ? sdesc(smem_u32(sB), BK * 128, 1024) : sdesc(smem_u32(sB), 16, 1024);
    constexpr uint64_t a_k = A_MN ? (2048 >> 4) : (32 >> 4);
    constexpr uint64_t b_k = B_MN ? (2048 >> 4) : (32 >> 4);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    int sslot = 0;
    uint32_t sphase = 0;
    while (true) {
      mbar_wait(&sfull[sslot], sphase);
      const int unit = ring[sslot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[sslot]);
      if (++sslot == kSchedDepth) {
        sslot = 0;
        sphase ^= 1;
      }
      if (unit >= nunits) break;
      const int split = unit / ntiles;
      const int kb_lo = split * nkb / nsplit, kb_hi = (split + 1) * nkb / nsplit;
      mbar_wait(&tempty[acc], acc_phase ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tbase + static_cast<uint32_t>(acc * 256);
      for (int kb = kb_lo; kb < kb_hi; ++kb) {
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        const uint64_t ad = a_desc0 + static_cast<uint64_t>(stage * (L::A_BYTES >> 4));
        const uint64_t bd = b_desc0 + static_cast<uint64_t>(stage * (L::B_BYTES >> 4));
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma_bf16(d_tmem, ad + k * a_k, bd + k * b_k, idesc, ((kb - kb_lo) | k) != 0 ? 1u : 0u);
          umma_commit(&empty[stage]);
        }
        __syncwarp();
        if (++stage == STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (elect_one()) umma_commit(&tfull[acc]);
      __syncwarp();
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  } else {
    // ===================== epilogue warps 2..5 =====================
    const int quarter = warp & 3;  // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    int acc = 0;
    uint32_t acc_phase = 0;
    int sslot = 0;
    uint32_t sphase = 0;
    while (true) {
      mbar_wait(&sfull[sslot], sphase);
      const int unit = ring[sslot];
      __syncwarp();
      if (lane == 0) mbar_arrive(&sempty[sslot]);
      if (++sslot == kSchedDepth) {
        sslot = 0;
        sphase ^= 1;
      }
      if (unit >= nunits) break;
      const int split = unit / ntiles, tile = unit - split * ntiles;
      int mb, nb;
      tile_coords(tile, num_m, num_n, sh.group, sh.group_n, mb, nb);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr =
          tbase + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * 256);
      epi.template apply<BN>(mb * BM, nb * BN, row, taddr, split);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512)
                 : "memory");
  }
}


// ---------------------------------------------------------------- the CTA-pair kernel
// (256 MB) x 256 output tile per cluster of 2 CTAs (cta_group::2, UMMA M=256 N=256): CTA r
// loads rows [128 MB r, 128 MB (r+1)) of the A tile and rows [128r, 128r+128) of the B tile
// (N-half); the leader (rank 0) issues the MMAs for both; each CTA's TMEM holds its 128 MB
// accumulator rows.  MB = 1: 256x256 tiles, two TMEM accumulators (epilogue of tile i
// overlaps the mainloop of tile i+1), 32 KB stages x 6.  MB = 2: 512x256 tiles (two MMAs per
// K step, one per 128-row block), one accumulator filling all 512 TMEM columns, 48 KB stages
// x 4 -- 27% less operand traffic per FLOP, for the long-K weight-gradient GEMM.
template <bool A_MN, bool B_MN, int STAGES, int MB = 1, int BN = 256>
struct Smem2 {
  static constexpr int A_BYTES = MB * BM * BK * 2;       // this CTA's 128 MB rows of A
  static constexpr int B_BYTES = (BN / 2) * BK * 2;      // this CTA's N-half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + (2 * STAGES + 4 + 2 * kSchedDepth) * 8 + 32 + 1024;
};

// MS: the persistent multi-step launch (TileShape::tsteps > 1).  Every multi-step branch is
// compiled only into the MS instantiations: a per-k-block test in the producer loop of the
// ordinary launches measured 7% on the backward step GEMM (profiles/r02_abb_final.txt).
template <bool A_MN, bool B_MN, int STAGES, int MB, int BN, class Epi, bool MS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc_gemm2_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap ta1,
                    const __grid_constant__ CUtensorMap tb0, const __grid_constant__ CUtensorMap tb1,
                    const TileShape sh, const Epi epi) {
  constexpr int TM = 2 * BM * MB;           // rows per cluster tile
  constexpr int NACC = MB == 1 ? 2 : 1;     // TMEM accumulator buffers (256 columns per block)
  static_assert(MB == 1 || MB == 2, "MB");
  static_assert(BN % 32 == 0 && BN <= 256, "pair UMMA N: multiple of 16 per CTA half");
  static_assert(!B_MN || (BN / 2) % 64 == 0, "MN-major B needs 64-wide panels per CTA half");
  using L = Smem2<A_MN, B_MN, STAGES, MB, BN>;
  TC_TRACE_BEGIN();
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;              // tile-index ring: filled
  uint64_t* sempty = sfull + kSchedDepth;    //                  consumed
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sempty + kSchedDepth);
  int* ring = reinterpret_cast<int*>(tslot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int nclusters = gridDim.x >> 1;
  const int num_m = (sh.M + TM - 1) / TM;
  const int num_n = (sh.N + BN - 1) / BN;
  const int ntiles = num_m * num_n;
  const int nsplit = sh.ksplit > 1 ? sh.ksplit : 1;
  // split-K: unit = split * ntiles + tile; multi-step: unit = step * ntiles + tile
  const int nunits = ntiles * (MS && sh.tsteps > 1 ? sh.tsteps : nsplit);

  if (threadIdx.x == 0) {
    prefetch_map(&ta0);
    prefetch_map(&tb0);
    if (sh.nkb1 > 0) {
      prefetch_map(&ta1);
      prefetch_map(&tb1);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);   // leader: one arrive.expect_tx for both CTAs' bytes
      mbar_init(&empty[s], 1);  // one multicast commit from the leader's MMA
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    for (int s = 0; s < kSchedDepth; ++s) {
      mbar_init(&sfull[s], 1);
      // leader copy: MMA warp + 4 + 4 epilogue warps + the follower's producer
      mbar_init(&sempty[s], 10);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  if (threadIdx.x == 0) TC_TRACE(1);

  if (warp == 0) {
    if (lane == 0) {
      // ===================== TMA producer (both CTAs) =====================
      // the leader's producer is the tile-scheduler fetcher for the pair; it publishes each
      // tile index into both CTAs' rings
      int stage = 0;
      uint32_t phase = 0;
      int sslot = 0;
      uint32_t sphase = 0;
      const uint32_t sempty_l0 = mapa_shared(smem_u32(&sempty[0]), 0);
      const uint32_t sfull_f0 = mapa_shared(smem_u32(&sfull[0]), 1);
      const uint32_t ring_f0 = mapa_shared(smem_u32(&ring[0]), 1);
      const int die = sh.die_split > 0 ? sh.sm_die[smid()] : 0;
      while (true) {
        int tile;
        if (leader) {
          mbar_wait(&sempty[sslot], sphase ^ 1);
          tile = sh.die_split > 0 ? sched_fetch_die(sh.sched, nunits, nclusters, die, sh.die_split)
                                  : sched_fetch(sh.sched, nunits, nclusters);
          ring[sslot] = tile;
          st_shared_cluster(ring_f0 + 4 * sslot, tile);
          mbar_arrive(&sfull[sslot]);
          mbar_arrive_cluster(sfull_f0 + 8 * sslot);
        } else {
          mbar_wait_cluster(&sfull[sslot], sphase);
          tile = ring[sslot];
          mbar_arrive_cluster(sempty_l0 + 8 * sslot);
        }
        if (++sslot == kSchedDepth) {
          sslot = 0;
          sphase ^= 1;
        }
        if (tile >= nunits) break;
        if (TC_SEL(tile, sslot == 1 && sphase == 0)) TC_TRACE(2);
        const UnitInfo ui = decode_unit<MS>(sh, tile, ntiles);
        const int kb_lo = ui.kb_lo, kb_hi = ui.kb_hi;
        int mb, nb;
        tile_coords(ui.tile, num_m, num_n, sh.group, sh.group_n, mb, nb);
        bool dep = MS && sh.tsteps > 1 && ui.split > 0;   // step s-1 of this row block must be done
        const int m_row = mb * TM + rank * BM * MB;  // this CTA's A rows
        const int n_row = nb * BN + rank * (BN / 2);  // this CTA's B rows (N-half)
        const unsigned int* drow =
            dep ? sh.ready + static_cast<int64_t>((ui.split - 1) * num_m + mb) * sh.dep_ld : nullptr;
        int oct = -1;          // fine mode: octet of ready groups last polled, and its bits
        uint32_t obits = 0;
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          // kx: the k-block in source order [source 0 | source 1].  dep_perm (the backward):
          // source 1 (dy_t, no dependency) first, then source 0's blocks in the order the
          // previous step's epilogues publish them (block q of every tile, then q + 1, ...)
          int kx = kb;
          if (MS && sh.src1_first && sh.tsteps > 1) {
            // multi-step backward: source 1 (dy_t, no dependency) while the previous step's
            // row block finishes, then source 0 (dz_{t+1})
            kx = kb < sh.nkb1 ? ui.nkb0 + kb : kb - sh.nkb1;
          } else if (MS && sh.dep_perm && sh.tsteps > 1) {
            if (kb < sh.nkb1) {
              kx = ui.nkb0 + kb;
            } else {
              const int i = (kb - sh.nkb1) / sh.dep_kpg, r = (kb - sh.nkb1) % sh.dep_kpg;
              const int tpr = sh.dep_ng / sh.epi_q;
              kx = sh.dep_kb + ((i % tpr) * sh.epi_q + i / tpr) * sh.dep_kpg + r;
            }
          }
          if (dep && kx >= sh.dep_kb && kx < ui.nkb0) {
            if (sh.dep_fine) {
              const int j = (kx - sh.dep_kb) / sh.dep_kpg;
              if (j < sh.dep_ng) {
                if ((j >> 3) != oct || !((obits >> (j & 7)) & 1u)) {
                  obits = wait_group(drow, j, 2u, true);
                  oct = j >> 3;
                }
              }
            } else {
              wait_ready(sh.ready + (ui.split - 1) * num_m + mb, 2u * num_n, true);
              if (TC_SEL(tile, false)) TC_TRACE(3);
              dep = false;
            }
          }
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fbar = mapa_shared(smem_u32(&full[stage]), 0);
          if (leader) mbar_expect_tx(&full[stage], 2 * L::STAGE_BYTES);
          const bool s1 = kx >= ui.nkb0;
          const int kk = (s1 ? kx - ui.nkb0 : kx + sh.kb_off) * BK;
          const CUtensorMap* ta = s1 ? &ta1 : &ta0;
          const CUtensorMap* tb = s1 ? &tb1 : &tb0;
          const int za = s1 ? ui.za1 : ui.za0;
          const int zb = s1 ? sh.zb1 : sh.zb0;
          uint8_t* a_dst = sA + stage * L::A_BYTES;
          uint8_t* b_dst = sB + stage * L::B_BYTES;
          if (!A_MN) {
            if (MS && sh.a_ilv) tma_load_4d_pair(ta, fbar, a_dst, kk, m_row >> 2, 0, za);
            else tma_load_3d_pair(ta, fbar, a_dst, kk, m_row, za);
          } else {
#pragma unroll
            for (int p = 0; p < 2 * MB; ++p)
              tma_load_3d_pair(ta, fbar, a_dst + p * (BK * 128), m_row + p * 64, kk, za);
          }
          if (!B_MN) {
            tma_load_3d_pair(tb, fbar, b_dst, kk, n_row, zb);
          } else {
#pragma unroll
            for (int p = 0; p < BN / 128; ++p)
              tma_load_3d_pair(tb, fbar, b_dst + p * (BK * 128), n_row + p * 64, kk, zb);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      TC_TRACE(10);
    }
  } else if (warp == 1) {
    if (leader) {
      // ===================== MMA issuer (leader): the warp waits, one lane issues ==========
      constexpr uint32_t idesc = idesc_bf16(2 * BM, BN, A_MN, B_MN);
      const uint64_t a_desc0 = A_MN ? sdesc(smem_u32(sA), BK * 128, 1024) : sdesc(smem_u32(sA), 16, 1024);
      const uint64_t b_desc0 = B_MN ? sdesc(smem_u32(sB), BK * 128, 1024) : sdesc(smem_u32(sB), 16, 1024);
      constexpr uint64_t a_k = A_MN ? (2048 >> 4) : (32 >> 4);
      constexpr uint64_t b_k = B_MN ? (2048 >> 4) : (32 >> 4);
      constexpr uint64_t a_blk = (BM * 128) >> 4;  // next 128-row block of A (both majors)
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int sslot = 0;
      uint32_t sphase = 0;
      while (true) {
        mbar_wait(&sfull[sslot], sphase);
        const int tile = ring[sslot];
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[sslot]);
        if (++sslot == kSchedDepth) {
          sslot = 0;
          sphase ^= 1;
        }
        if (tile >= nunits) break;
        const UnitInfo ui = decode_unit<MS>(sh, tile, ntiles);
        const int kb_lo = ui.kb_lo, kb_hi = ui.kb_hi;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tbase + static_cast<uint32_t>(acc * 256);
        for (int kb = kb_lo; kb < kb_hi; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          if (lane == 0 && kb == kb_lo && TC_SEL(tile, sslot == 1 && sphase == 0)) TC_TRACE(4);
          const uint64_t ad = a_desc0 + static_cast<uint64_t>(stage * (L::A_BYTES >> 4));
          const uint64_t bd = b_desc0 + static_cast<uint64_t>(stage * (L::B_BYTES >> 4));
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
#pragma unroll
              for (int b = 0; b < MB; ++b)
                umma_bf16_pair(d_tmem + b * 256, ad + b * a_blk + k * a_k, bd + k * b_k, idesc,
                               ((kb - kb_lo) | k) != 0 ? 1u : 0u);
            umma_commit_pair(&empty[stage]);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit_pair(&tfull[acc]);
        __syncwarp();
        if (lane == 0 && TC_SEL(tile, sslot == 1 && sphase == 0)) TC_TRACE(5);
        if (++acc == NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (lane == 0) TC_TRACE(11);
    }
  } else {
    // ===================== epilogue warps 2..5 (both CTAs) =====================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t tempty_leader0 = mapa_shared(smem_u32(&tempty[0]), 0);
    const uint32_t sempty_l0 = mapa_shared(smem_u32(&sempty[0]), 0);
    int acc = 0;
    uint32_t acc_phase = 0;
    int sslot = 0;
    uint32_t sphase = 0;
    while (true) {
      if (leader) mbar_wait(&sfull[sslot], sphase);
      else mbar_wait_cluster(&sfull[sslot], sphase);
      const int tile = ring[sslot];
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(sempty_l0 + 8 * sslot);
      if (++sslot == kSchedDepth) {
        sslot = 0;
        sphase ^= 1;
      }
      if (tile >= nunits) break;
      const int split = tile / ntiles;
      int mb, nb;
      tile_coords(tile - split * ntiles, num_m, num_n, sh.group, sh.group_n, mb, nb);
      if (MS && sh.tsteps > 1 && split > 0) {
        // the epilogue reads the previous step's cell state (c / dc) of this row block
        if (lane == 0) {
          if (sh.dep_fine) {
            const unsigned int* drow =
                sh.ready + static_cast<int64_t>((split - 1) * num_m + mb) * sh.dep_ld;
            for (int q = 0; q < sh.epi_q; ++q) wait_group(drow, nb * sh.epi_q + q, 2u, false);
          } else {
            wait_ready(sh.ready + (split - 1) * num_m + mb, 2u * num_n, false);
          }
        }
        __syncwarp();
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      if (threadIdx.x == 64 && TC_SEL(tile, sslot == 1 && sphase == 0)) TC_TRACE(6);
      if (lane == 0 && TC_SEL(tile, sslot == 1 && sphase == 0)) TC_TRACE(16 + quarter);
      const uint32_t taddr =
          tbase + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * 256);
      bool done = false;
      constexpr int FB = FineBlocks<Epi>::v;
      if constexpr (MB == 1 && FB > 0) {
        if (MS && sh.tsteps > 1 && sh.dep_fine) {
          // publish each block as soon as it is stored: the next step's k-blocks of that block
          // (and the block's next-step epilogue) may start before the whole tile is done.
          // epi_q = 1: the tile is one block (forward: 256 gate columns = 64 units); epi_q =
          // BN / 64: 64 output columns per block (backward: dh columns = hidden units)
          unsigned int* drow = sh.ready + static_cast<int64_t>(split * num_m + mb) * sh.dep_ld;
          constexpr int QW = BN / FB;   // output columns per block
#pragma unroll 1
          for (int q = 0; q < FB; ++q) {
            epi.template apply<QW>(mb * TM + rank * BM, nb * BN + q * QW, row, taddr + q * QW,
                                   split);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            if (threadIdx.x == 64) {
              __threadfence();
              atomicAdd(drow + nb * FB + q, 1u);
            }
          }
          done = true;
        }
      }
      if (!done) {
#pragma unroll 1
        for (int b = 0; b < MB; ++b)
          epi.template apply<BN>(mb * TM + rank * BM * MB + b * BM, nb * BN, row, taddr + b * 256,
                                 split);
      }
      if (threadIdx.x == 64 && TC_SEL(tile, sslot == 1 && sphase == 0)) TC_TRACE(7);
      if (lane == 0 && TC_SEL(tile, sslot == 1 && sphase == 0)) TC_TRACE(20 + quarter);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_leader0 + acc * 8);
      if (MS && sh.tsteps > 1 && !sh.dep_fine) {
        // this CTA's half of the tile is stored: publish it to the next step (cumulative
        // fence by one thread after the epilogue warps' barrier)
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) {
          __threadfence();
          atomicAdd(sh.ready + split * num_m + mb, 1u);
        }
      }
      if (++acc == NACC) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) TC_TRACE(12 + quarter);
  }

  if (threadIdx.x == 0) TC_TRACE(8);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512)
                 : "memory");
    if (lane == 0) TC_TRACE(9);
  }
}

// ---------------------------------------------------------------- 2 CTA pairs, B multicast
// Cluster of 4 = two CTA pairs stacked along M (m-tiles 2u and 2u+1, the same N tile).  Each
// pair runs the pair kernel's 256x256 tile (K-major A and B, double-buffered accumulators),
// but the two pairs share the B operand: every CTA loads 64 of its pair-half's 128 B rows and
// multicasts them to the same-rank CTA of the other pair, so the L2 supplies each B tile once
// per cluster (25% fewer L2->SM operand bytes per FLOP).  Completion is tracked per CTA (plain
// multicast: each destination's own full barrier); the follower of each pair forwards its
// stage completion to the pair leader, whose MMA waits for both; a stage is released when
// both pairs' MMAs committed it (commit multicast to all 4 CTAs, count 2).
template <int STAGES>
struct SmemMC {
  static constexpr int A_BYTES = BM * BK * 2;          // this CTA's 128 A rows
  static constexpr int B_BYTES = 128 * BK * 2;         // this CTA's 128-row N-half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + (3 * STAGES + 4 + 2 * kSchedDepth) * 8 + 32 + 1024;
};
__device__ __forceinline__ void tma_load_3d_mc(const CUtensorMap* map, uint64_t* bar, void* dst,
                                               int c0, int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2),
      "h"(mask)
      : "memory");
}
// 2-SM multicast: data lands at the same offset in every CTA of mask; complete_tx is counted on
// the mbarrier at bar's offset in each destination CTA's pair leader (bar: a cluster address)
__device__ __forceinline__ void tma_load_3d_pair_mc(const CUtensorMap* map, uint32_t bar_cluster,
                                                    void* dst, int c0, int c1, int c2,
                                                    uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2),
      "h"(mask)
      : "memory");
}
__device__ __forceinline__ void umma_commit_mask(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)), "h"(mask)
      : "memory");
}

template <int STAGES, class Epi>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(kThreads, 1)
    tc_gemm2mc_kernel(const __grid_constant__ CUtensorMap ta0, const __grid_constant__ CUtensorMap tb0,
                      const TileShape sh, const Epi epi) {
  constexpr int BN = 256, TM = 2 * BM;     // per-pair tile 256 x 256
  using L = SmemMC<STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);   // this CTA's bytes
  uint64_t* fullP = full + STAGES;                                   // leader: follower's done
  uint64_t* empty = fullP + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + kSchedDepth;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sempty + kSchedDepth);
  int* ring = reinterpret_cast<int*>(tslot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t pair = rank >> 1, prank = rank & 1, pl = rank & ~1u;
  const int nclusters = gridDim.x >> 2;
  const int num_m = (sh.M + TM - 1) / TM;          // 256-row tiles
  const int num_mu = (num_m + 1) / 2;              // units: pairs of m-tiles
  const int num_n = (sh.N + BN - 1) / BN;
  const int nunits = num_mu * num_n;
  const int nkb = sh.nkb0;

  if (threadIdx.x == 0) {
    prefetch_map(&ta0);
    prefetch_map(&tb0);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);    // pair leader: one arrive.expect_tx for both CTAs' bytes
      mbar_init(&fullP[s], 1);   // (unused with 2-SM multicast)
      mbar_init(&empty[s], 2);   // one commit from each pair's MMA
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);  // 4 epilogue warps x 2 CTAs of the pair (leader's copy)
    }
    for (int s = 0; s < kSchedDepth; ++s) {
      mbar_init(&sfull[s], 1);
      // rank 0's copy: rank0 MMA + 4 epi; ranks 1,3 producer + 4 epi; rank 2 producer + MMA
      // + 4 epi
      mbar_init(&sempty[s], 21);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t sempty_c0 = mapa_shared(smem_u32(&sempty[0]), 0);

  // reads the next unit from this CTA's ring (rank 0's own copy, the others' written remotely)
  auto next_unit = [&](int& sslot, uint32_t& sphase, bool arrive) -> int {
    if (rank == 0) mbar_wait(&sfull[sslot], sphase);
    else mbar_wait_cluster(&sfull[sslot], sphase);
    const int u = ring[sslot];
    if (arrive) mbar_arrive_cluster(sempty_c0 + 8 * sslot);
    if (++sslot == kSchedDepth) {
      sslot = 0;
      sphase ^= 1;
    }
    return u;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ===================== TMA producer (all 4 CTAs); rank 0 also fetches units ==========
      int stage = 0;
      uint32_t phase = 0;
      int sslot = 0;
      uint32_t sphase = 0;
      const uint16_t bmask = (uint16_t)((1u << prank) | (1u << (prank + 2)));
      while (true) {
        int unit;
        if (rank == 0) {
          mbar_wait(&sempty[sslot], sphase ^ 1);
          unit = sched_fetch(sh.sched, nunits, nclusters);
          ring[sslot] = unit;
          mbar_arrive(&sfull[sslot]);
#pragma unroll
          for (uint32_t r = 1; r < 4; ++r) {
            st_shared_cluster(mapa_shared(smem_u32(&ring[sslot]), r), unit);
            mbar_arrive_cluster(mapa_shared(smem_u32(&sfull[sslot]), r));
          }
          if (++sslot == kSchedDepth) {
            sslot = 0;
            sphase ^= 1;
          }
        } else {
          unit = next_unit(sslot, sphase, true);
        }
        if (unit >= nunits) break;
        int mu, nb;
        tile_coords(unit, num_mu, num_n, sh.group, sh.group_n, mu, nb);
        const int m_row = (2 * mu + (int)pair) * TM + (int)prank * BM;
        const int n_row = nb * BN + (int)prank * 128 + (int)pair * 64;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fbar = mapa_shared(smem_u32(&full[stage]), pl);
          if (prank == 0) mbar_expect_tx(&full[stage], 2 * L::STAGE_BYTES);
          const int kk = (kb + sh.kb_off) * BK;
          tma_load_3d_pair(&ta0, fbar, sA + stage * L::A_BYTES, kk, m_row, sh.za0);
          tma_load_3d_pair_mc(&tb0, fbar, sB + stage * L::B_BYTES + pair * (64 * 128), kk,
                              n_row, sh.zb0, bmask);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    int sslot = 0;
    uint32_t sphase = 0;
    int stage = 0;
    uint32_t phase = 0;
    if (prank == 0) {
      // ===================== MMA issuer (pair leaders) =====================
      constexpr uint32_t idesc = idesc_bf16(2 * BM, BN, false, false);
      const uint64_t a_desc0 = sdesc(smem_u32(sA), 16, 1024);
      const uint64_t b_desc0 = sdesc(smem_u32(sB), 16, 1024);
      constexpr uint64_t a_k = 32 >> 4, b_k = 32 >> 4;
      const uint16_t pmask = (uint16_t)(0x3u << (2 * pair));
      int acc = 0;
      uint32_t acc_phase = 0;
      while (true) {
        const int unit = next_unit(sslot, sphase, lane == 0);
        __syncwarp();
        if (unit >= nunits) break;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tbase + static_cast<uint32_t>(acc * 256);
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = a_desc0 + static_cast<uint64_t>(stage * (L::A_BYTES >> 4));
          const uint64_t bd = b_desc0 + static_cast<uint64_t>(stage * (L::B_BYTES >> 4));
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
              umma_bf16_pair(d_tmem, ad + k * a_k, bd + k * b_k, idesc, (kb | k) != 0 ? 1u : 0u);
            umma_commit_mask(&empty[stage], (uint16_t)0xF);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit_mask(&tfull[acc], pmask);
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===================== epilogue warps 2..5 (all CTAs) =====================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t tempty_pl0 = mapa_shared(smem_u32(&tempty[0]), pl);
    int acc = 0;
    uint32_t acc_phase = 0;
    int sslot = 0;
    uint32_t sphase = 0;
    while (true) {
      const int unit = next_unit(sslot, sphase, lane == 0);
      __syncwarp();
      if (unit >= nunits) break;
      int mu, nb;
      tile_coords(unit, num_mu, num_n, sh.group, sh.group_n, mu, nb);
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const uint32_t taddr =
          tbase + (static_cast<uint32_t>(quarter * 32) << 16) + static_cast<uint32_t>(acc * 256);
      epi.template apply<BN>((2 * mu + (int)pair) * TM + (int)prank * BM, nb * BN, row, taddr, 0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_pl0 + acc * 8);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512)
                 : "memory");
  }
}

// ---------------------------------------------------------------- 2 CTA pairs, A multicast
// Weight-gradient variant: a cluster of 4 = two CTA pairs stacked along N (n-tiles 2u and
// 2u+1 of the same 512-row M tile, MB = 2, MN-major A and B).  The pairs share the A operand
// (the dZ panel): CTA (pair p, rank r) loads A panels {2p, 2p+1} of its 256 rows and
// multicasts them to the same-rank CTA of the other pair, so the L2 supplies each A tile once
// per cluster: per pair and K block 256 + 256 instead of 512 + 256 operand rows (-33% L2->SM
// bytes per FLOP).  Barriers as tc_gemm2mc_kernel: completion counted on each destination
// pair's leader, a stage released when both pairs' MMAs committed it.
template <int STAGES>
struct SmemMCA {
  static constexpr int A_BYTES = 2 * BM * BK * 2;      // this CTA's 256 A rows (4 panels)
  static constexpr int B_BYTES = 128 * BK * 2;         // this CTA's 128-row N-half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr int TOTAL = BAR_OFF + (2 * STAGES + 4 + 2 * kSchedDepth) * 8 + 32 + 1024;
};

template <int STAGES, class Epi>
__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(kThreads, 1)
    tc_gemm2mca_kernel(const __grid_constant__ CUtensorMap ta0,
                       const __grid_constant__ CUtensorMap tb0, const TileShape sh,
                       const Epi epi) {
  constexpr int BN = 256, TM = 4 * BM;     // per-pair tile 512 x 256
  using L = SmemMCA<STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * L::A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* sfull = tempty + 2;
  uint64_t* sempty = sfull + kSchedDepth;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sempty + kSchedDepth);
  int* ring = reinterpret_cast<int*>(tslot + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const uint32_t pair = rank >> 1, prank = rank & 1, pl = rank & ~1u;
  const int nclusters = gridDim.x >> 2;
  const int num_m = (sh.M + TM - 1) / TM;          // 512-row tiles
  const int num_n = (sh.N + BN - 1) / BN;
  const int num_nu = (num_n + 1) / 2;              // units: pairs of n-tiles
  const int nunits = num_m * num_nu;
  const int nkb = sh.nkb0;

  if (threadIdx.x == 0) {
    prefetch_map(&ta0);
    prefetch_map(&tb0);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);    // pair leader: one arrive.expect_tx for both CTAs' bytes
      mbar_init(&empty[s], 2);   // one commit from each pair's MMA
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 8);  // 4 epilogue warps x 2 CTAs of the pair (leader's copy)
    }
    for (int s = 0; s < kSchedDepth; ++s) {
      mbar_init(&sfull[s], 1);
      // rank 0's copy: rank0 MMA + 4 epi; ranks 1,3 producer + 4 epi; rank 2 producer + MMA
      // + 4 epi
      mbar_init(&sempty[s], 21);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tbase = *tslot;
  const uint32_t sempty_c0 = mapa_shared(smem_u32(&sempty[0]), 0);

  auto next_unit = [&](int& sslot, uint32_t& sphase, bool arrive) -> int {
    if (rank == 0) mbar_wait(&sfull[sslot], sphase);
    else mbar_wait_cluster(&sfull[sslot], sphase);
    const int u = ring[sslot];
    if (arrive) mbar_arrive_cluster(sempty_c0 + 8 * sslot);
    if (++sslot == kSchedDepth) {
      sslot = 0;
      sphase ^= 1;
    }
    return u;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ===================== TMA producer (all 4 CTAs); rank 0 also fetches units ==========
      int stage = 0;
      uint32_t phase = 0;
      int sslot = 0;
      uint32_t sphase = 0;
      const uint16_t amask = (uint16_t)((1u << prank) | (1u << (prank + 2)));
      while (true) {
        int unit;
        if (rank == 0) {
          mbar_wait(&sempty[sslot], sphase ^ 1);
          unit = sched_fetch(sh.sched, nunits, nclusters);
          ring[sslot] = unit;
          mbar_arrive(&sfull[sslot]);
#pragma unroll
          for (uint32_t r = 1; r < 4; ++r) {
            st_shared_cluster(mapa_shared(smem_u32(&ring[sslot]), r), unit);
            mbar_arrive_cluster(mapa_shared(smem_u32(&sfull[sslot]), r));
          }
          if (++sslot == kSchedDepth) {
            sslot = 0;
            sphase ^= 1;
          }
        } else {
          unit = next_unit(sslot, sphase, true);
        }
        if (unit >= nunits) break;
        int mb, nu;
        tile_coords(unit, num_m, num_nu, sh.group, sh.group_n, mb, nu);
        const int m_row = mb * TM + (int)prank * 2 * BM;           // this CTA's 256 A rows
        const int n_row = (2 * nu + (int)pair) * BN + (int)prank * 128;
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t fbar = mapa_shared(smem_u32(&full[stage]), pl);
          if (prank == 0) mbar_expect_tx(&full[stage], 2 * L::STAGE_BYTES);
          const int kk = (kb + sh.kb_off) * BK;
          uint8_t* a_dst = sA + stage * L::A_BYTES;
          uint8_t* b_dst = sB + stage * L::B_BYTES;
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int p = 2 * (int)pair + q;                        // my share of the panels
            tma_load_3d_pair_mc(&ta0, fbar, a_dst + p * (BK * 128), m_row + p * 64,
                                kk, sh.za0, amask);
          }
#pragma unroll
          for (int p = 0; p < 2; ++p)
            tma_load_3d_pair(&tb0, fbar, b_dst + p * (BK * 128), n_row + p * 64, kk, sh.zb0);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    int sslot = 0;
    uint32_t sphase = 0;
    int stage = 0;
    uint32_t phase = 0;
    if (prank == 0) {
      // ===================== MMA issuer (pair leaders) =====================
      constexpr uint32_t idesc = idesc_bf16(2 * BM, BN, true, true);
      const uint64_t a_desc0 = sdesc(smem_u32(sA), BK * 128, 1024);
      const uint64_t b_desc0 = sdesc(smem_u32(sB), BK * 128, 1024);
      constexpr uint64_t a_k = 2048 >> 4, b_k = 2048 >> 4;
      constexpr uint64_t a_blk = (BM * 128) >> 4;   // next 128-row block of A
      const uint16_t pmask = (uint16_t)(0x3u << (2 * pair));
      uint32_t acc_phase = 0;
      while (true) {
        const int unit = next_unit(sslot, sphase, lane == 0);
        __syncwarp();
        if (unit >= nunits) break;
        mbar_wait(&tempty[0], acc_phase ^ 1);
        tc_fence_after();
        for (int kb = 0; kb < nkb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = a_desc0 + static_cast<uint64_t>(stage * (L::A_BYTES >> 4));
          const uint64_t bd = b_desc0 + static_cast<uint64_t>(stage * (L::B_BYTES >> 4));
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k)
#pragma unroll
              for (int b = 0; b < 2; ++b)
                umma_bf16_pair(tbase + b * 256, ad + b * a_blk + k * a_k, bd + k * b_k, idesc,
                               (kb | k) != 0 ? 1u : 0u);
            umma_commit_mask(&empty[stage], (uint16_t)0xF);
          }
          __syncwarp();
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit_mask(&tfull[0], pmask);
        __syncwarp();
        acc_phase ^= 1;
      }
    }
  } else {
    // ===================== epilogue warps 2..5 (all CTAs) =====================
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t tempty_pl0 = mapa_shared(smem_u32(&tempty[0]), pl);
    uint32_t acc_phase = 0;
    int sslot = 0;
    uint32_t sphase = 0;
    while (true) {
      const int unit = next_unit(sslot, sphase, lane == 0);
      __syncwarp();
      if (unit >= nunits) break;
      int mb, nu;
      tile_coords(unit, num_m, num_nu, sh.group, sh.group_n, mb, nu);
      mbar_wait(&tfull[0], acc_phase);
      tc_fence_after();
      const uint32_t taddr = tbase + (static_cast<uint32_t>(quarter * 32) << 16);
#pragma unroll 1
      for (int b = 0; b < 2; ++b)
        epi.template apply<BN>(mb * TM + (int)prank * 2 * BM + b * BM, (2 * nu + (int)pair) * BN,
                               row, taddr + b * 256, 0);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(tempty_pl0);
      acc_phase ^= 1;
    }
  }

  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) {
    __syncwarp();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(512)
                 : "memory");
  }
}

// ---------------------------------------------------------------- epilogues

// Plain fp32 store: out[m*ldc + n] for m < M, n < N.
struct EpiStoreF32 {
  float* out;
  int64_t ldc;
  int M, N;
  int64_t split_stride;  // elements between split-K partial outputs
  int accumulate;        // 1: out += acc (K-chunked launches after the first)
  template <int BN>
  __device__ __forceinline__ void apply(int m_base, int n_base, int row, uint32_t taddr,
                                        int split) const {
    const int m = m_base + row;
    const bool vec = (N % 4 == 0) && (ldc % 4 == 0);
#pragma unroll 1
    for (int c = 0; c < BN / 16; ++c) {
      float v[16];
      tmem_ld16(taddr + c * 16, v);
      const int n0 = n_base + c * 16;
      if (m >= M || n0 >= N) continue;
      float* dst = out + split * split_stride + static_cast<int64_t>(m) * ldc + n0;
      if (vec && n0 + 16 <= N) {
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          if (accumulate) {
            const float4 p = d4[q];
            o.x += p.x;
            o.y += p.y;
            o.z += p.z;
            o.w += p.w;
          }
          d4[q] = o;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (n0 + i < N) dst[i] = accumulate ? dst[i] + v[i] : v[i];
      }
    }
  }
};

// EpiStoreF32 whose final values also go to the DP owners' staging (fused exchange, push
// mode; a separate type so the default launches keep the lean epilogue)
struct EpiStoreF32Dp {
  float* out;
  int64_t ldc;
  int M, N;
  int64_t split_stride;  // elements between split-K partial outputs
  int accumulate;        // 1: out += acc (K-chunked launches after the first)
  // final values also pushed to the DP owners' staging (fused exchange, push mode): element
  // (m, n) is theta element dp_base + m * ldc + n; dp.world == 0: off
  ppo::DpStage dp{};
  int64_t dp_base = 0;
  template <int BN>
  __device__ __forceinline__ void apply(int m_base, int n_base, int row, uint32_t taddr,
                                        int split) const {
    const int m = m_base + row;
    const bool vec = (N % 4 == 0) && (ldc % 4 == 0);
#pragma unroll 1
    for (int c = 0; c < BN / 16; ++c) {
      float v[16];
      tmem_ld16(taddr + c * 16, v);
      const int n0 = n_base + c * 16;
      if (m >= M || n0 >= N) continue;
      const int64_t e0 = static_cast<int64_t>(m) * ldc + n0;
      float* dst = out + split * split_stride + e0;
      if (vec && n0 + 16 <= N) {
        float4* d4 = reinterpret_cast<float4*>(dst);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          float4 o = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          if (accumulate) {
            const float4 p = d4[q];
            o.x += p.x;
            o.y += p.y;
            o.z += p.z;
            o.w += p.w;
          }
          d4[q] = o;
          // over NVLink to the owner of these 4 elements (shards are multiples of 64)
          if (dp.world) *reinterpret_cast<float4*>(dp.slot(dp_base + e0 + 4 * q)) = o;
        }
      } else {
#pragma unroll
        for (int i = 0; i < 16; ++i)
          if (n0 + i < N) {
            const float o = accumulate ? dst[i] + v[i] : v[i];
            dst[i] = o;
            if (dp.world) *dp.slot(dp_base + e0 + i) = o;
          }
      }
    }
  }
};

// Transposed fp32 store: out[split][n][m] (ldc = row stride of the [N][M] output).  Lane =
// row m, so each store instruction writes 32 consecutive m of one column n (coalesced).
// Used by the skinny inference GEMMs (weights = M, batch = N) so consumers read per batch row.
struct EpiStoreF32T {
  float* out;
  int64_t ldc;
  int M, N;
  int64_t split_stride;
  template <int BN>
  __device__ __forceinline__ void apply(int m_base, int n_base, int row, uint32_t taddr,
                                        int split) const {
    const int m = m_base + row;
    float* base = out + split * split_stride + m;
#pragma unroll 1
    for (int c = 0; c < BN / 16; ++c) {
      float v[16];
      tmem_ld16(taddr + c * 16, v);
      const int n0 = n_base + c * 16;
      if (m >= M || n0 >= N) continue;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (n0 + i < N) base[static_cast<int64_t>(n0 + i) * ldc] = v[i];
    }
  }
};

__device__ __forceinline__ void load_bf16x16(const __nv_bfloat16* p, float (&v)[16]) {
  const uint4* q = reinterpret_cast<const uint4*>(p);
  uint4 a = q[0], b = q[1];
  const __nv_bfloat162* h0 = reinterpret_cast<const __nv_bfloat162*>(&a);
  const __nv_bfloat162* h1 = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 f0 = __bfloat1622float2(h0[i]);
    float2 f1 = __bfloat1622float2(h1[i]);
    v[2 * i] = f0.x;
    v[2 * i + 1] = f0.y;
    v[8 + 2 * i] = f1.x;
    v[8 + 2 * i + 1] = f1.y;
  }
}
__device__ __forceinline__ void store_bf16x16(__nv_bfloat16* p, const float (&v)[16]) {
  uint4 a, b;
  __nv_bfloat162* h0 = reinterpret_cast<__nv_bfloat162*>(&a);
  __nv_bfloat162* h1 = reinterpret_cast<__nv_bfloat162*>(&b);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    h0[i] = __floats2bfloat162_rn(v[2 * i], v[2 * i + 1]);
    h1[i] = __floats2bfloat162_rn(v[8 + 2 * i], v[8 + 2 * i + 1]);
  }
  // one 32-byte sector: a single 256-bit store (sm_100)
  asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(a.x), "r"(a.y),
               "r"(a.z), "r"(a.w), "r"(b.x), "r"(b.y), "r"(b.z), "r"(b.w)
               : "memory");
}
// 16 floats = two 32-byte sectors: two 256-bit loads / stores (sm_100)
__device__ __forceinline__ void load_f32x16(const float* p, float (&v)[16]) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
    asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(v[8 * h]), "=f"(v[8 * h + 1]), "=f"(v[8 * h + 2]), "=f"(v[8 * h + 3]),
                   "=f"(v[8 * h + 4]), "=f"(v[8 * h + 5]), "=f"(v[8 * h + 6]), "=f"(v[8 * h + 7])
                 : "l"(p + 8 * h));
}
__device__ __forceinline__ void store_f32x16(float* p, const float (&v)[16]) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
    asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p + 8 * h),
                 "f"(v[8 * h]), "f"(v[8 * h + 1]), "f"(v[8 * h + 2]), "f"(v[8 * h + 3]),
                 "f"(v[8 * h + 4]), "f"(v[8 * h + 5]), "f"(v[8 * h + 6]), "f"(v[8 * h + 7])
                 : "memory");
}

// LSTM forward step t (oracle O4).  Tile = 128 sequences x 256 gate rows = 4 gates of 64
// hidden units (gate-interleaved W rows), so the whole cell update is tile-local.
struct EpiLstmFwd {
  static constexpr int kFineBlocks = 1;   // a tile = 4 gates x 64 units: one unit block
  __nv_bfloat16* h_out;   // XH[t+1] + D  (row stride ldxh)
  int64_t ldxh;
  const float* c_prev;    // C[t]   [B][H]
  float* c_out;           // C[t+1] [B][H]
  __nv_bfloat16* gates;   // G[t]   [B][4H], interleaved like the accumulator columns
  int B, H;
  int64_t sx, sc, sg;     // multi-step launch: per-step element strides of XH, C and G
  int ilv;                // TMEM lane r holds row 4 (r % 32) + r / 32 (TileShape::a_ilv)
  template <int BN>
  __device__ __forceinline__ void apply(int m_base, int n_base, int row, uint32_t taddr,
                                        int step) const {
    static_assert(BN == 256, "cell tile holds 4 gates x 64 units");
    __nv_bfloat16* const h_out = this->h_out + step * sx;
    const float* const c_prev = this->c_prev + step * sc;
    float* const c_out = this->c_out + step * sc;
    __nv_bfloat16* const gates = this->gates + step * sg;
    const int m = m_base + (ilv ? (row & 31) * 4 + (row >> 5) : row);
    const bool ok = m < B;
    const int64_t G4 = 4 * static_cast<int64_t>(H);
#pragma unroll 1
    for (int u0 = 0; u0 < 64; u0 += 16) {
      float zi[16], zf[16], zg[16], zo[16];
      tmem_ld16(taddr + 0 + u0, zi);
      tmem_ld16(taddr + 64 + u0, zf);
      tmem_ld16(taddr + 128 + u0, zg);
      tmem_ld16(taddr + 192 + u0, zo);
      if (!ok) continue;
      const int j0 = n_base / 4 + u0;
      float cp[16], c[16], h[16];
      load_f32x16(c_prev + static_cast<int64_t>(m) * H + j0, cp);
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        float i, f, g, o;
        cell_fwd_tc(zi[e], zf[e], zg[e], zo[e], cp[e], i, f, g, o, c[e], h[e]);
        zi[e] = i;
        zf[e] = f;
        zg[e] = g;
        zo[e] = o;
      }
      store_f32x16(c_out + static_cast<int64_t>(m) * H + j0, c);
      store_bf16x16(h_out + static_cast<int64_t>(m) * ldxh + j0, h);
      __nv_bfloat16* gp = gates + static_cast<int64_t>(m) * G4 + n_base + u0;
      store_bf16x16(gp + 0, zi);
      store_bf16x16(gp + 64, zf);
      store_bf16x16(gp + 128, zg);
      store_bf16x16(gp + 192, zo);
    }
  }
};

// LSTM backward step t (oracle O8).  Accumulator = dh_t = dz_{t+1} W_h + dy_t W_o for 256
// hidden units; the cell backward reads the saved gates of step t and overwrites them with dz_t.
// Chunks of 8 units; the saved activations of chunk c+1 are loaded (raw 16-byte vectors) while
// chunk c computes, so the HBM latency of the loads overlaps the math.
struct BwdRaw {
  uint4 g[4];            // gates i, f, g, o: 8 bf16 each
  float4 ct[2], cp[2], dc[2];
};
// 32-byte (one sector) loads and stores of 8 floats: sm_100's 256-bit LDG/STG
__device__ __forceinline__ void ld_f32x8(const float* p, float4 (&v)[2]) {
  asm volatile("ld.global.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0].x), "=f"(v[0].y), "=f"(v[0].z), "=f"(v[0].w), "=f"(v[1].x),
                 "=f"(v[1].y), "=f"(v[1].z), "=f"(v[1].w)
               : "l"(p));
}
__device__ __forceinline__ void st_f32x8(float* p, const float4 (&v)[2]) {
  asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "f"(v[0].x),
               "f"(v[0].y), "f"(v[0].z), "f"(v[0].w), "f"(v[1].x), "f"(v[1].y), "f"(v[1].z),
               "f"(v[1].w)
               : "memory");
}
__device__ __forceinline__ void bwd_load(BwdRaw& r, const __nv_bfloat16* gp, const float* ct,
                                         const float* cp, const float* dc) {
#pragma unroll
  for (int q = 0; q < 4; ++q) r.g[q] = *reinterpret_cast<const uint4*>(gp + q * 64);
  ld_f32x8(ct, r.ct);   // 8 units of c_t, c_{t-1}, dc: one full 32-byte sector each
  ld_f32x8(cp, r.cp);
  if (dc) {
    ld_f32x8(dc, r.dc);
  } else {
    r.dc[0] = make_float4(0.f, 0.f, 0.f, 0.f);
    r.dc[1] = r.dc[0];
  }
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  __syncwarp();
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

// TAIL: stop at the last chunk inside H (no TMEM loads of a last N tile's columns past H) --
// only in the multi-step instantiation: any change to this loop in the per-step kernel moved
// the backward step GEMM at B = 38,400 by 2-3% (profiles/r02_nch_ab.txt, r02_nch2_ab.txt)
template <bool TAIL>
struct EpiLstmBwdT {
  static constexpr int kFineBlocks = 4;   // a tile = 256 units of dh: four unit blocks
  __nv_bfloat16* gz;      // G[t]: gates in, dz out  [B][4H]
  const float* c_t;       // C[t+1]
  const float* c_prev;    // C[t]
  float* dc;              // [B][H] carry (in/out)
  int B, H;
  int first;              // 1: t = T-1, the incoming carry is zero (not read; no memset)
  int exp;                // PPO_EXPERIMENTS builds only (timing A/B, wrong results):
                          // bit0 skip the saved-activation loads, bit1 skip the stores
  int64_t sc, sg;         // multi-step launch (step s = time T-1-s): per-step strides of C, G
  int ilv;                // TMEM lane r holds row 4 (r % 32) + r / 32 (TileShape::a_ilv)
  template <int BN>
  __device__ __forceinline__ void apply(int m_base, int n_base, int row, uint32_t taddr,
                                        int step) const {
    __nv_bfloat16* const gz = this->gz + step * sg;
    const float* const c_t = this->c_t + step * sc;
    const float* const c_prev = this->c_prev + step * sc;
    const bool first = this->first && step == 0;
    constexpr int CW = 8;  // units per chunk
    const int m = m_base + (ilv ? (row & 31) * 4 + (row >> 5) : row);
    const bool ok = m < B;
    const int64_t G4 = 4 * static_cast<int64_t>(H);
    const int nch = max(0, min(BN, H - n_base)) / CW;
    const __nv_bfloat16* grow = gz + static_cast<int64_t>(m) * G4;
    const int64_t crow = static_cast<int64_t>(m) * H + n_base;
    auto goff = [&](int cc) {
      const int j0 = n_base + cc * CW;
      return (j0 >> 6) * 256 + (j0 & 63);
    };
    // the saved activations of chunk cc + 1 are loaded while chunk cc computes (two chunks
    // ahead measured 2% slower in the step at B = 38,400: profiles/r02_ab_bwd_ahead.txt)
    BwdRaw cur, nxt;
    const float* dcin = first ? nullptr : dc;
#ifdef PPO_EXPERIMENTS
    const bool no_ld = exp & 1, no_st = exp & 2;
#else
    constexpr bool no_ld = false, no_st = false;
#endif
    if (no_ld) cur = BwdRaw{};
    auto load_chunk = [&](BwdRaw& r, int cc) {
      const int64_t o = crow + cc * CW;
      bwd_load(r, grow + goff(cc), c_t + o, c_prev + o, dcin ? dcin + o : nullptr);
    };
    if (ok && !no_ld && nch > 0) load_chunk(cur, 0);
#pragma unroll 1
    for (int cc = 0; cc < BN / CW; ++cc) {
      if constexpr (TAIL) {
        if (cc >= nch) break;
      }
      float dh[8];
      tmem_ld8(taddr + cc * CW, dh);
      if constexpr (!TAIL) {
        if (cc >= nch) continue;
      }
      if (ok && cc + 1 < nch && !no_ld) load_chunk(nxt, cc + 1);
      if (ok) {
        // in place: each 32-bit gate word holds units (2w, 2w+1); dz overwrites the gates
        float* ct = reinterpret_cast<float*>(cur.ct);
        float* cp = reinterpret_cast<float*>(cur.cp);
        float* dcv = reinterpret_cast<float*>(cur.dc);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          float z[4][2];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const uint32_t u = reinterpret_cast<const uint32_t*>(&cur.g[q])[w];
            z[q][0] = __uint_as_float(u << 16);
            z[q][1] = __uint_as_float(u & 0xFFFF0000u);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int e = 2 * w + h;
            float a, b, c, d, dn;
            cell_bwd(dh[e], dcv[e], z[0][h], z[1][h], z[2][h], z[3][h], ct[e], cp[e], a, b, c,
                     d, dn, true);
            z[0][h] = a;
            z[1][h] = b;
            z[2][h] = c;
            z[3][h] = d;
            dcv[e] = dn;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const __nv_bfloat162 pk = __floats2bfloat162_rn(z[q][0], z[q][1]);
            reinterpret_cast<uint32_t*>(&cur.g[q])[w] = *reinterpret_cast<const uint32_t*>(&pk);
          }
        }
        if (!no_st) {
          __nv_bfloat16* gp = gz + static_cast<int64_t>(m) * G4 + goff(cc);
#pragma unroll
          for (int q = 0; q < 4; ++q) *reinterpret_cast<uint4*>(gp + q * 64) = cur.g[q];
          st_f32x8(dc + crow + cc * CW, cur.dc);
        } else if (cur.dc[0].x == 1234.5f) {   // keep the math live
          dc[crow] = cur.dc[1].y + __uint_as_float(cur.g[0].x);
        }
      }
      if (!no_ld) cur = nxt;
    }
  }
};
using EpiLstmBwd = EpiLstmBwdT<false>;
using EpiLstmBwdTail = EpiLstmBwdT<true>;

}  // namespace tc
}  // namespace ppo
