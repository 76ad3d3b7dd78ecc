// api.cu -- the extern "C" boundary of libppo5.so (include/ppo5.h): argument checking,
// workspace layout and the composition of each hot-path call from the kernels.
#include <math.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"

#include <nvtx3/nvToolsExt.h>

namespace ppo {

static thread_local std::string g_err;
void set_error(const std::string& msg) { g_err = msg; }
int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* what) {
  g_err = std::string(what) + ": " + cudaGetErrorString(e);
  return PPO_E_CUDA;
}

// ---- tracing ------------------------------------------------------------------------------
namespace {
struct ProfRec {
  std::string tag;
  cudaEvent_t a, b;
};
struct Prof {
  std::mutex mu;
  bool on = false;
  std::vector<ProfRec> recs;
  std::vector<int> open;  // indices of records awaiting their end event
  std::vector<cudaEvent_t> pool;
  cudaEvent_t get() {
    if (!pool.empty()) {
      cudaEvent_t e = pool.back();
      pool.pop_back();
      return e;
    }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
  }
};
Prof& prof() {
  static Prof p;
  return p;
}
}  // namespace

void prof_begin(const char* tag, cudaStream_t s) {
  nvtxRangePushA(tag);   // NVTX range per library launch (no-op without an attached tool)
  Prof& P = prof();
  if (!P.on) return;
  std::lock_guard<std::mutex> g(P.mu);
  ProfRec r{tag, P.get(), P.get()};
  cudaEventRecord(r.a, s);
  P.recs.push_back(r);
  P.open.push_back((int)P.recs.size() - 1);
}
void prof_end(cudaStream_t s) {
  nvtxRangePop();
  Prof& P = prof();
  if (!P.on) return;
  std::lock_guard<std::mutex> g(P.mu);
  if (P.open.empty()) return;
  cudaEventRecord(P.recs[P.open.back()].b, s);
  P.open.pop_back();
}

int num_sms() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
    return 148;
  return n;
}

int check_dims(const ppo_dims* d, Shape* s) {
  if (!d) return fail(PPO_E_ARG, "dims is NULL");
  if (d->D <= 0 || d->H <= 0 || d->T <= 0 || d->D % 64 || d->H % 64)
    return fail(PPO_E_SHAPE, "D and H must be positive multiples of 64, T >= 1");
  if (d->n_heads < 1 || d->n_heads > PPO_MAX_HEADS)
    return fail(PPO_E_SHAPE, "n_heads must be in [1, 8]");
  if (d->precision != PPO_PREC_BF16 && d->precision != PPO_PREC_FP32)
    return fail(PPO_E_ARG, "unknown precision");
  s->D = d->D;
  s->H = d->H;
  s->T = d->T;
  s->G4 = 4LL * d->H;
  s->Kx = (int64_t)d->D + d->H + 64;
  s->Ko = (int64_t)d->H + 64;
  s->n_heads = d->n_heads;
  s->head_off[0] = 0;
  for (int k = 0; k < d->n_heads; ++k) {
    if (d->head_sizes[k] <= 0) return fail(PPO_E_SHAPE, "head sizes must be positive");
    s->head_off[k + 1] = s->head_off[k] + d->head_sizes[k];
  }
  if (d->head_sizes[0] > 64) return fail(PPO_E_SHAPE, "primary head must have <= 64 actions");
  if (d->n_aux_win < 0 || d->n_aux_win > 1 || d->n_aux_rank < 0 || d->n_aux_rank > 32 ||
      d->n_aux_bld < 0 || d->n_aux_bld > 64)
    return fail(PPO_E_SHAPE, "aux heads: n_aux_win in {0,1}, n_aux_rank <= 32, n_aux_bld <= 64");
  if (!(d->aux_win_trunk >= 0.f) || !(d->aux_win_trunk < 1e30f))
    return fail(PPO_E_ARG, "aux_win_trunk must be finite and >= 0");
  s->vcol = s->head_off[d->n_heads];
  s->n_win = d->n_aux_win;
  s->n_rank = d->n_aux_rank;
  s->n_bld = d->n_aux_bld;
  s->n_aux = s->n_win + s->n_rank + s->n_bld;
  s->win_trunk = d->aux_win_trunk;
  s->win_pass = s->n_win && d->aux_win_trunk > 0.f;
  s->A = s->vcol + 1 + s->n_aux;
  s->A_pass = s->vcol + 1 + (s->win_pass ? 1 : 0);
  s->bf16 = d->precision == PPO_PREC_BF16;
  if (s->bf16 && (s->A * 2) % 16)
    return fail(PPO_E_SHAPE, "bf16 path needs A*2 to be a multiple of 16 bytes (TMA stride)");
  return PPO_OK;
}

static size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

WsLayout ws_layout(const Shape& s, int64_t B) {
  const size_t esz = s.bf16 ? 2 : 4;
  WsLayout L{};
  size_t off = 0;
  L.xh = off;
  off = align_up(off + (size_t)(s.T + 1) * B * s.Kx * esz, 1024);
  L.g = off;
  off = align_up(off + (size_t)s.T * B * s.G4 * esz, 1024);
  L.c = off;
  off = align_up(off + (size_t)(s.T + 1) * B * s.H * 4, 1024);
  L.dc = off;
  off = align_up(off + (size_t)B * s.H * 4, 1024);
  L.raw = off;
  if (!s.bf16) off = align_up(off + (size_t)B * s.G4 * 4, 1024);
  L.splitk = off;  // split-K partials of dW_o (bf16 path)
  if (s.bf16) off = align_up(off + (size_t)kMaxSplitK * s.A * s.Ko * 4, 1024);
  L.sched = off;   // tile-scheduler counters of this workspace's GEMMs, then the per-step
                   // ready counters of a multi-step launch (T x ceil(B / 256) x ready_ld(H))
  L.ready = off + kSchedBytes;
  off = align_up(L.ready + ready_bytes(s.T, B, s.H), 1024);
  L.total = off;
  return L;
}

static int param_layout(const Shape& s, ppo_param_layout* o) {
  o->Kx = s.Kx;
  o->Ko = s.Ko;
  o->A = s.A;
  o->off_wxh = 0;
  o->n_wxh = s.G4 * s.Kx;
  o->off_wo = o->n_wxh;
  o->n_wo = s.A * s.Ko;
  o->n_total = o->n_wxh + o->n_wo;
  return PPO_OK;
}

static int need(const void* p, const char* name) {
  if (!p) return fail(PPO_E_ARG, std::string(name) + " is NULL");
  if (!aligned(p, 16)) return fail(PPO_E_ALIGN, std::string(name) + " is not 16-byte aligned");
  return PPO_OK;
}
#define NEED(p)                          \
  do {                                   \
    int _r = need((p), #p);              \
    if (_r) return _r;                   \
  } while (0)

int check_tc_device() {
  int dev = 0, major = 0;
  PPO_CUDA_CHECK(cudaGetDevice(&dev));
  PPO_CUDA_CHECK(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
  if (major != 10) return fail(PPO_E_UNSUPPORTED, "bf16 tcgen05 path needs an sm_100 device");
  return PPO_OK;
}

}  // namespace ppo

using namespace ppo;

// comm.cu: the push-mode staging of an attached comm (C++ linkage, library-internal)
const ppo::DpStage* ppo_comm_dp_stage(const ppo_comm* c);
size_t ppo_comm_dp_n(const ppo_comm* c);

extern "C" {

const char* ppo_last_error(void) { return g_err.c_str(); }
const char* ppo_version(void) { return "libppo5 0.1 (sm_100a; tcgen05 bf16 + SIMT fp32 paths)"; }

int ppo_get_param_layout(const ppo_dims* dims, ppo_param_layout* out) {
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (!out) return fail(PPO_E_ARG, "out is NULL");
  return param_layout(s, out);
}

int ppo_pack_params(const ppo_dims* dims, const float* Wx, const float* Wh, const float* b,
                    const float* Wo, const float* bo, float* theta, ppo_stream_t st) {
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (!Wx || !Wh || !b || !Wo || !bo || !theta) return fail(PPO_E_ARG, "NULL pointer");
  ppo_param_layout L;
  param_layout(s, &L);
  return launch_pack_params(s, Wx, Wh, b, Wo, bo, theta, L.n_wxh, L.n_total, (cudaStream_t)st);
}

int ppo_unpack_params(const ppo_dims* dims, const float* theta, float* Wx, float* Wh, float* b,
                      float* Wo, float* bo, ppo_stream_t st) {
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (!Wx || !Wh || !b || !Wo || !bo || !theta) return fail(PPO_E_ARG, "NULL pointer");
  ppo_param_layout L;
  param_layout(s, &L);
  return launch_unpack_params(s, theta, Wx, Wh, b, Wo, bo, L.n_wxh, (cudaStream_t)st);
}

int ppo_cast_bf16(const float* src, uint16_t* dst, size_t n, ppo_stream_t st) {
  if (n == 0) return PPO_OK;
  if (!src || !dst) return fail(PPO_E_ARG, "NULL pointer");
  return launch_cast_bf16(src, dst, n, (cudaStream_t)st);
}

int ppo_gae_scratch_bytes(int64_t R, int64_t L, size_t* bytes) {
  if (R < 0 || L < 0) return fail(PPO_E_SHAPE, "R and L must be >= 0");
  if (!bytes) return fail(PPO_E_ARG, "bytes is NULL");
  *bytes = (R == 0 || L == 0) ? 0 : gae_scratch_bytes(R, L);
  return PPO_OK;
}

int ppo_gae(const float* rew, const float* val, const uint8_t* done, int64_t R, int64_t L,
            float gamma, float lam, int32_t seq_T, float* adv, float* ret, void* scratch,
            size_t scratch_bytes, ppo_stream_t st) {
  if (R < 0 || L < 0) return fail(PPO_E_SHAPE, "R and L must be >= 0");
  if (R == 0 || L == 0) return PPO_OK;
  if (!rew || !val || !done || !adv || !ret) return fail(PPO_E_ARG, "NULL pointer");
  if (seq_T < 0 || (seq_T > 0 && L % seq_T)) return fail(PPO_E_SHAPE, "L must be a multiple of seq_T");
  if (!(gamma >= 0.f && gamma <= 1.f && lam >= 0.f && lam <= 1.f))
    return fail(PPO_E_ARG, "gamma and lam must be in [0, 1]");
  const size_t need = gae_scratch_bytes(R, L);
  if (need > 0 && (!scratch || scratch_bytes < need || !aligned(scratch, 16)))
    return fail(PPO_E_ARG, "long rollouts need ppo_gae_scratch_bytes() of 16-byte aligned scratch");
  return launch_gae(rew, val, done, R, L, gamma, lam, seq_T, adv, ret, scratch, (cudaStream_t)st);
}

int lstm_ws_bytes(const ppo_dims* dims, int64_t B, size_t* bytes) {
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (B < 1) return fail(PPO_E_SHAPE, "B must be >= 1");
  if (!bytes) return fail(PPO_E_ARG, "bytes is NULL");
  *bytes = ws_layout(s, B).total;
  return PPO_OK;
}

static int fwd_impl(const ppo_dims* dims, const void* w, const void* x, const float* h0,
                    const float* c0, int64_t B, void* ws, size_t ws_bytes, float* out,
                    const cudaEvent_t* x_ready, ppo_stream_t st_) {
  cudaStream_t st = (cudaStream_t)st_;
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (B < 1) return fail(PPO_E_SHAPE, "B must be >= 1");
  if (s.bf16 && B * s.T > (int64_t)INT32_MAX / 2) return fail(PPO_E_SHAPE, "T*B too large");
  NEED(w);
  NEED(out);
  if (x) {
    NEED(h0);
    NEED(c0);
    if (!aligned(x, 16)) return fail(PPO_E_ALIGN, "x is not 16-byte aligned");
  }
  if (!ws || !aligned(ws, 1024)) return fail(PPO_E_ALIGN, "ws must be 1024-byte aligned");
  WsLayout L = ws_layout(s, B);
  if (ws_bytes < L.total) return fail(PPO_E_ARG, "workspace too small");
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  float* C = reinterpret_cast<float*>(wsb + L.c);
  // x == NULL: x already in the workspace (lstm_ws_x / ppo_copy_x: pack h0, c0 and the pad
  // columns; or ppo_gather, which also placed h0/c0: nothing to do)
  if (x) {
    if ((rc = launch_pack_x(s, B, x, h0, c0, wsb + L.xh, C, st))) return rc;
  } else if (h0 || c0) {
    if (!h0 || !c0 || !aligned(h0, 16) || !aligned(c0, 16))
      return fail(PPO_E_ARG, "h0 and c0 must both be given (16-byte aligned)");
    if ((rc = launch_pack_state(s, B, h0, c0, wsb + L.xh, C, st))) return rc;
  }
  if (s.bf16) {
    if ((rc = check_tc_device())) return rc;
    return tc_forward(s, B, w, ws, out, x_ready, st);
  }
  // ---- SIMT fp32 reference path
  const float* W = static_cast<const float*>(w);
  const float* Wo = W + s.G4 * s.Kx;
  float* XH = reinterpret_cast<float*>(wsb + L.xh);
  float* G = reinterpret_cast<float*>(wsb + L.g);
  float* raw = reinterpret_cast<float*>(wsb + L.raw);
  for (int64_t t = 0; t < s.T; ++t) {
    if (x_ready && x_ready[t]) PPO_CUDA_CHECK(cudaStreamWaitEvent(st, x_ready[t], 0));
    SimtOp a{{XH + t * B * s.Kx, nullptr}, {s.Kx, 0}, {B, 0}, {s.Kx, 0}, s.Kx, false};
    SimtOp b{{W, nullptr}, {s.Kx, 0}, {s.G4, 0}, {s.Kx, 0}, s.Kx, false};
    if ((rc = launch_simt_gemm(a, b, B, s.G4, s.Kx, raw, s.G4, st))) return rc;
    if ((rc = launch_simt_cell_fwd(s, B, raw, C + t * B * s.H, C + (t + 1) * B * s.H,
                                   XH + (t + 1) * B * s.Kx + s.D, s.Kx, G + t * B * s.G4, st)))
      return rc;
  }
  SimtOp a{{XH + B * s.Kx + s.D, nullptr}, {s.Kx, 0}, {s.T * B, 0}, {s.Ko, 0}, s.Ko, false};
  SimtOp b{{Wo, nullptr}, {s.Ko, 0}, {s.A, 0}, {s.Ko, 0}, s.Ko, false};
  return launch_simt_gemm(a, b, s.T * B, s.A, s.Ko, out, s.A, st);
}

int lstm_bptt_fwd(const ppo_dims* dims, const void* w, const void* x, const float* h0,
                  const float* c0, int64_t B, void* ws, size_t ws_bytes, float* out,
                  ppo_stream_t st) {
  return fwd_impl(dims, w, x, h0, c0, B, ws, ws_bytes, out, nullptr, st);
}

int lstm_bptt_fwd_ev(const ppo_dims* dims, const void* w, const float* h0, const float* c0,
                     int64_t B, void* ws, size_t ws_bytes, float* out,
                     void* const* x_ready, ppo_stream_t st) {
  return fwd_impl(dims, w, nullptr, h0, c0, B, ws, ws_bytes, out,
                  reinterpret_cast<const cudaEvent_t*>(x_ready), st);
}

int ppo_copy_x_slice(const ppo_dims* dims, int64_t B, int32_t t, const void* src,
                     int64_t src_ld, void* ws, size_t ws_bytes, ppo_stream_t st) {
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (B < 1 || t < 0 || t >= s.T) return fail(PPO_E_SHAPE, "need B >= 1 and 0 <= t < T");
  if (!src || !ws) return fail(PPO_E_ARG, "NULL pointer");
  if (src_ld < s.D) return fail(PPO_E_ARG, "src_ld < D");
  WsLayout L = ws_layout(s, B);
  if (ws_bytes < L.total) return fail(PPO_E_ARG, "workspace too small");
  const size_t esz = s.bf16 ? 2 : 4;
  ProfScope _prof("copy_x", (cudaStream_t)st);
  PPO_CUDA_CHECK(cudaMemcpy2DAsync(static_cast<uint8_t*>(ws) + L.xh + (size_t)t * B * s.Kx * esz,
                                   s.Kx * esz, src, src_ld * esz, s.D * esz, B,
                                   cudaMemcpyDefault, (cudaStream_t)st));
  return PPO_OK;
}

int lstm_ws_x(const ppo_dims* dims, int64_t B, void* ws, void** x, int64_t* ld) {
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (B < 1) return fail(PPO_E_SHAPE, "B must be >= 1");
  if (!ws || !x || !ld) return fail(PPO_E_ARG, "NULL pointer");
  *x = static_cast<uint8_t*>(ws) + ws_layout(s, B).xh;
  *ld = s.Kx;
  return PPO_OK;
}

int ppo_copy_x(const ppo_dims* dims, int64_t B, const void* src, int64_t src_ld, void* ws,
               size_t ws_bytes, ppo_stream_t st) {
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (B < 1) return fail(PPO_E_SHAPE, "B must be >= 1");
  if (!src || !ws) return fail(PPO_E_ARG, "NULL pointer");
  if (src_ld < s.D) return fail(PPO_E_ARG, "src_ld < D");
  WsLayout L = ws_layout(s, B);
  if (ws_bytes < L.total) return fail(PPO_E_ARG, "workspace too small");
  const size_t esz = s.bf16 ? 2 : 4;
  ProfScope _prof("copy_x", (cudaStream_t)st);
  PPO_CUDA_CHECK(cudaMemcpy2DAsync(static_cast<uint8_t*>(ws) + L.xh, s.Kx * esz, src,
                                   src_ld * esz, s.D * esz, s.T * B, cudaMemcpyDefault,
                                   (cudaStream_t)st));
  return PPO_OK;
}

int ppo_loss_grad(const ppo_dims* dims, const float* out, const int32_t* act,
                  const uint8_t* head_on, const uint8_t* avail, const float* logp_old,
                  const float* adv, const float* ret, const uint8_t* valid,
                  const float* aux_label, int64_t B, const ppo_loss_cfg* cfg, void* dout,
                  float* logp, float* stats, ppo_stream_t st) {
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (B < 1) return fail(PPO_E_SHAPE, "B must be >= 1");
  if (!out || !act || !head_on || !avail || !logp_old || !adv || !ret || !cfg || !dout || !stats)
    return fail(PPO_E_ARG, "NULL pointer");
  if (s.n_aux && !aux_label) return fail(PPO_E_ARG, "aux heads need aux_label");
  LossParams p{};
  p.N = s.T * B;
  p.A = (int)s.A;
  p.vcol = s.vcol;
  p.n_win = s.n_win;
  p.n_rank = s.n_rank;
  p.n_aux = s.n_aux;
  p.c_win = cfg->c_win;
  p.c_rank = cfg->c_rank;
  p.c_bld = cfg->c_bld;
  p.win_scale = s.win_pass ? s.win_trunk : 1.f;
  p.A_pad = (int)((s.A + 31) / 32 * 32);
  p.nh = s.n_heads;
  for (int k = 0; k <= s.n_heads; ++k) p.off[k] = s.head_off[k];
  p.clip_eps = cfg->clip_eps;
  p.c_v = cfg->c_v;
  p.c_e = cfg->c_e;
  const double denom = cfg->denom > 0 ? cfg->denom : (double)p.N;
  p.inv_denom = (float)(1.0 / denom);
  if ((size_t)p.A_pad * 8 * sizeof(float) > 48 * 1024) return fail(PPO_E_SHAPE, "A too large");
  if (s.A > 6 * 128) return fail(PPO_E_SHAPE, "loss kernel supports A <= 768");
  return launch_loss(p, s.bf16, out, act, head_on, avail, logp_old, adv, ret, valid, aux_label,
                     dout, logp, stats, (cudaStream_t)st);
}

int lstm_bptt_bwd_dp(const ppo_dims* dims, const void* w, void* ws, size_t ws_bytes,
                     const void* dout, int64_t B, float* grad, ppo_comm* comm,
                     ppo_stream_t st_) {
  if (!comm) return fail(PPO_E_ARG, "comm is NULL");
  const ppo::DpStage* dp = ppo_comm_dp_stage(comm);
  if (!dp) return fail(PPO_E_ARG, "comm has no attached dp buffers (ppo_dp_attach, world > 1)");
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (!s.bf16) return fail(PPO_E_UNSUPPORTED, "push-mode dp exchange needs the bf16 path");
  if (s.win_pass) return fail(PPO_E_UNSUPPORTED, "push-mode dp exchange: no win-head trunk scale");
  if (ppo_comm_dp_n(comm) != (size_t)(s.G4 * s.Kx + s.A * s.Ko))
    return fail(PPO_E_SHAPE, "attached dp length differs from this model's theta");
  if (B < 1) return fail(PPO_E_SHAPE, "B must be >= 1");
  NEED(w);
  NEED(dout);
  NEED(grad);
  if (!ws || !aligned(ws, 1024)) return fail(PPO_E_ALIGN, "ws must be 1024-byte aligned");
  if (ws_bytes < ws_layout(s, B).total) return fail(PPO_E_ARG, "workspace too small");
  if ((rc = check_tc_device())) return rc;
  return tc_backward(s, B, w, ws, dout, grad, (cudaStream_t)st_, dp);
}

int lstm_bptt_bwd(const ppo_dims* dims, const void* w, void* ws, size_t ws_bytes,
                  const void* dout, int64_t B, float* grad, ppo_stream_t st_) {
  return lstm_bptt_bwd_ev(dims, w, ws, ws_bytes, dout, B, grad, nullptr, st_);
}

int lstm_bptt_bwd_ev(const ppo_dims* dims, const void* w, void* ws, size_t ws_bytes,
                     const void* dout, int64_t B, float* grad, void* wxh_ready_ev,
                     ppo_stream_t st_) {
  cudaStream_t st = (cudaStream_t)st_;
  cudaEvent_t wxh_ready = static_cast<cudaEvent_t>(wxh_ready_ev);
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (B < 1) return fail(PPO_E_SHAPE, "B must be >= 1");
  NEED(w);
  NEED(dout);
  NEED(grad);
  if (!ws || !aligned(ws, 1024)) return fail(PPO_E_ALIGN, "ws must be 1024-byte aligned");
  WsLayout L = ws_layout(s, B);
  if (ws_bytes < L.total) return fail(PPO_E_ARG, "workspace too small");
  if (s.bf16) {
    if ((rc = check_tc_device())) return rc;
    return tc_backward(s, B, w, ws, dout, grad, st, nullptr, wxh_ready);
  }
  // ---- SIMT fp32 reference path
  uint8_t* wsb = static_cast<uint8_t*>(ws);
  const float* W = static_cast<const float*>(w);
  const float* Wo = W + s.G4 * s.Kx;
  const float* dY = static_cast<const float*>(dout);
  float* XH = reinterpret_cast<float*>(wsb + L.xh);
  float* G = reinterpret_cast<float*>(wsb + L.g);
  float* C = reinterpret_cast<float*>(wsb + L.c);
  float* dc = reinterpret_cast<float*>(wsb + L.dc);
  float* raw = reinterpret_cast<float*>(wsb + L.raw);
  PPO_CUDA_CHECK(cudaMemsetAsync(dc, 0, B * s.H * sizeof(float), st));
  for (int64_t t = s.T - 1; t >= 0; --t) {
    const bool last = t == s.T - 1;
    const float* dYt = dY + t * B * s.A;
    SimtOp a, b;
    int64_t K;
    // only the first A_pass output columns reach the LSTM (stop_gradient aux heads, Q26)
    if (last) {  // dh_{T-1} = dy_{T-1} W_o only
      a = SimtOp{{dYt, nullptr}, {s.A, 0}, {B, 0}, {s.A_pass, 0}, s.A_pass, false};
      b = SimtOp{{Wo, nullptr}, {s.Ko, 0}, {s.H, 0}, {s.A_pass, 0}, s.A_pass, true};
      K = s.A_pass;
    } else {     // dh_t = dz_{t+1} W_h + dy_t W_o
      a = SimtOp{{G + (t + 1) * B * s.G4, dYt}, {s.G4, s.A}, {B, B}, {s.G4, s.A_pass}, s.G4,
                 false};
      b = SimtOp{{W + s.D, Wo}, {s.Kx, s.Ko}, {s.H, s.H}, {s.G4, s.A_pass}, s.G4, true};
      K = s.G4 + s.A_pass;
    }
    if ((rc = launch_simt_gemm(a, b, B, s.H, K, raw, s.H, st))) return rc;
    if ((rc = launch_simt_cell_bwd(s, B, raw, G + t * B * s.G4, C + (t + 1) * B * s.H,
                                   C + t * B * s.H, dc, st)))
      return rc;
  }
  const int64_t rows = s.T * B;
  {
    SimtOp a{{G, nullptr}, {s.G4, 0}, {s.G4, 0}, {rows, 0}, rows, true};
    SimtOp b{{XH, nullptr}, {s.Kx, 0}, {s.Kx, 0}, {rows, 0}, rows, true};
    if ((rc = launch_simt_gemm(a, b, s.G4, s.Kx, rows, grad, s.Kx, st))) return rc;
  }
  if (wxh_ready) PPO_CUDA_CHECK(cudaEventRecord(wxh_ready, st));
  {
    SimtOp a{{dY, nullptr}, {s.A, 0}, {s.A, 0}, {rows, 0}, rows, true};
    SimtOp b{{XH + B * s.Kx + s.D, nullptr}, {s.Kx, 0}, {s.Ko, 0}, {rows, 0}, rows, true};
    if ((rc = launch_simt_gemm(a, b, s.A, s.Ko, rows, grad + s.G4 * s.Kx, s.Ko, st))) return rc;
  }
  if (s.win_pass)  // dout's win column carries win_trunk x the gradient (Q26)
    return launch_scale(grad + s.G4 * s.Kx + (int64_t)(s.vcol + 1) * s.Ko, s.Ko,
                        1.f / s.win_trunk, st);
  return PPO_OK;
}

int lstm_input_grad(const ppo_dims* dims, const void* w, const void* ws, size_t ws_bytes,
                    int64_t B, float* dx, ppo_stream_t st_) {
  cudaStream_t st = (cudaStream_t)st_;
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (B < 1) return fail(PPO_E_SHAPE, "B must be >= 1");
  NEED(w);
  NEED(dx);
  if (!ws || !aligned(ws, 1024)) return fail(PPO_E_ALIGN, "ws must be 1024-byte aligned");
  WsLayout L = ws_layout(s, B);
  if (ws_bytes < L.total) return fail(PPO_E_ARG, "workspace too small");
  void* wsm = const_cast<void*>(ws);
  if (s.bf16) {
    if ((rc = check_tc_device())) return rc;
    return tc_input_grad(s, B, w, wsm, dx, st);
  }
  const float* G = reinterpret_cast<const float*>(static_cast<const uint8_t*>(ws) + L.g);
  const int64_t rows = s.T * B;
  SimtOp a{{G, nullptr}, {s.G4, 0}, {rows, 0}, {s.G4, 0}, s.G4, false};
  SimtOp b{{static_cast<const float*>(w), nullptr}, {s.Kx, 0}, {s.D, 0}, {s.G4, 0}, s.G4, true};
  ProfScope _prof("input_grad", st);
  return launch_simt_gemm(a, b, rows, s.D, s.G4, dx, s.D, st);
}

int adam_step(float* p, uint16_t* p_bf16, const float* g, float* m, float* v, size_t n,
              int64_t t, double lr, double b1, double b2, double eps, double clip_sigma,
              ppo_stream_t st) {
  if (n == 0) return PPO_OK;
  NEED(p);
  NEED(g);
  NEED(m);
  NEED(v);
  if (p_bf16 && !aligned(p_bf16, 16)) return fail(PPO_E_ALIGN, "p_bf16 is not 16-byte aligned");
  if (t < 1) return fail(PPO_E_ARG, "t must be >= 1");
  if (!(b1 >= 0.0 && b1 < 1.0 && b2 >= 0.0 && b2 < 1.0)) return fail(PPO_E_ARG, "bad betas");
  const AdamParams ap = make_adam_params(t, lr, b1, b2, eps, clip_sigma);
  return launch_adam(p, p_bf16, g, m, v, n, ap, (cudaStream_t)st);
}

int adam_step_ctr(float* p, uint16_t* p_bf16, const float* g, float* m, float* v, size_t n,
                  int64_t* ctr, double lr, double b1, double b2, double eps, double clip_sigma,
                  ppo_stream_t st) {
  NEED(ctr);
  if (!aligned(ctr, 16)) return fail(PPO_E_ALIGN, "ctr is not 16-byte aligned");
  if (n == 0) return PPO_OK;
  NEED(p);
  NEED(g);
  NEED(m);
  NEED(v);
  if (p_bf16 && !aligned(p_bf16, 16)) return fail(PPO_E_ALIGN, "p_bf16 is not 16-byte aligned");
  if (!(b1 >= 0.0 && b1 < 1.0 && b2 >= 0.0 && b2 < 1.0)) return fail(PPO_E_ARG, "bad betas");
  const AdamParams ap = make_adam_params(1, lr, b1, b2, eps, clip_sigma);   // alpha: device
  return launch_adam(p, p_bf16, g, m, v, n, ap, (cudaStream_t)st, ctr, lr);
}

int ppo_prof_start(void) {
  Prof& P = prof();
  std::lock_guard<std::mutex> g(P.mu);
  for (auto& r : P.recs) {
    P.pool.push_back(r.a);
    P.pool.push_back(r.b);
  }
  P.recs.clear();
  P.open.clear();
  P.on = true;
  return PPO_OK;
}

int ppo_prof_stop(ppo_prof_entry* out, int32_t max_entries, int32_t* n_out) {
  Prof& P = prof();
  std::lock_guard<std::mutex> g(P.mu);
  P.on = false;
  std::map<std::string, std::pair<int, double>> agg;
  std::vector<std::string> order;
  for (auto& r : P.recs) {
    PPO_CUDA_CHECK(cudaEventSynchronize(r.b));
    float ms = 0.f;
    PPO_CUDA_CHECK(cudaEventElapsedTime(&ms, r.a, r.b));
    auto it = agg.find(r.tag);
    if (it == agg.end()) {
      order.push_back(r.tag);
      agg[r.tag] = {1, ms};
    } else {
      it->second.first += 1;
      it->second.second += ms;
    }
  }
  int n = 0;
  for (auto& tag : order) {
    if (out && n < max_entries) {
      memset(out[n].name, 0, sizeof(out[n].name));
      strncpy(out[n].name, tag.c_str(), sizeof(out[n].name) - 1);
      out[n].launches = agg[tag].first;
      out[n].total_ms = agg[tag].second;
    }
    ++n;
  }
  if (n_out) *n_out = n;
  return PPO_OK;
}

// ---- testing hook (not part of the step): one tcgen05 GEMM, see tc_path.cu -------------
int ppo_test_tc_gemm(int mode, const uint16_t* A, const uint16_t* B, float* C, int M, int N, int K,
                     ppo_stream_t st) {
  if (!A || !B || !C || M <= 0 || N <= 0 || K <= 0) return fail(PPO_E_ARG, "bad test GEMM args");
  int rc = check_tc_device();
  if (rc) return rc;
  return tc_test_gemm(mode, A, B, C, M, N, K, (cudaStream_t)st);
}

}  // extern "C"
