/*
 * ppo5.h -- C ABI of libppo5.so: the data-parallel PPO optimizer step of OpenAI Five
 * (arXiv 1912.06680), B200-native (sm_100a).
 *
 * Citations: P:n = PAPER.md line n [section]; Qn / On = DESIGN.md readings / oracle
 * equations.  The step (§3.2):
 *     ppo_gae -> lstm_bptt_fwd -> ppo_loss_grad -> lstm_bptt_bwd -> grad_allreduce -> adam_step
 *
 * Conventions (all calls):
 *   - Pointers are DEVICE pointers unless marked (host).  The caller (PyTorch) owns every
 *     buffer; the library never allocates in a hot call.  Buffers must be 16-byte aligned
 *     (PPO_E_ALIGN otherwise); workspaces 1024-byte aligned.
 *   - Calls are asynchronous on the given stream (NULL = legacy default stream).  Host-
 *     checkable errors return immediately with a message in ppo_last_error()
 *     (thread-local).  Data errors found on the device (non-finite loss, unavailable taken
 *     action, empty availability row) set bits in stats[PPO_STAT_FLAGS]; the caller checks
 *     them after synchronising and aborts the step.
 *   - Results are deterministic for fixed inputs and world size (no float atomics).
 *   - A workspace (lstm_ws_bytes / ppo_infer_ws_bytes) serves one call at a time: it holds
 *     the saved activations and the tile-scheduler counters of the GEMMs launched on it.
 *     Calls in flight concurrently (two streams, two optimizers) must use distinct
 *     workspaces; nothing else in the library is shared between streams.
 *   - bf16 values are passed as uint16_t bit patterns.
 *   - Empty inputs: elementwise calls (ppo_gae with R*L = 0, adam_step with n = 0) are
 *     no-ops returning PPO_OK before any pointer check; the LSTM and loss calls need
 *     B >= 1 (PPO_E_SHAPE otherwise).
 */
#ifndef PPO5_H
#define PPO5_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* ppo_stream_t; /* == cudaStream_t */

enum {
  PPO_OK = 0,
  PPO_E_ARG = -1,         /* bad pointer / value */
  PPO_E_SHAPE = -2,       /* unsupported or inconsistent sizes */
  PPO_E_ALIGN = -3,       /* misaligned pointer */
  PPO_E_CUDA = -4,        /* CUDA runtime/driver error (message has the CUDA string) */
  PPO_E_NCCL = -5,        /* NCCL error */
  PPO_E_UNSUPPORTED = -6  /* e.g. no sm_100 device for the tcgen05 path */
};

enum { PPO_PREC_BF16 = 0, PPO_PREC_FP32 = 1 };

#define PPO_MAX_HEADS 8

/* Network shape.  D = LSTM input width (DESIGN Q1: 4032), H = hidden units (4096),
 * T = TBPTT length (16), heads = factorised action heads (P:303-368:
 * 30,4,189,189,81,81,81).  A = sum(head_sizes) + 1 (value).
 * D and H must be multiples of 64; T >= 1; 1 <= n_heads <= 8; head_sizes[0] <= 64
 * (the primary head carries the availability mask).
 * precision: PPO_PREC_BF16 = tcgen05 tensor cores, bf16 operands, fp32 accumulate;
 *            PPO_PREC_FP32 = SIMT fp32 reference path (parity 1e-4). */
typedef struct {
  int32_t D, H, T;
  int32_t n_heads;
  int32_t head_sizes[PPO_MAX_HEADS];
  int32_t precision;
  /* NEXT-4 auxiliary heads (DESIGN Q24-Q27), appended after the value output:
   * n_aux_win in {0,1} logistic win probability, n_aux_rank in [0,32] softmax net-worth
   * rank, n_aux_bld in [0,64] logistic enemy-building predictions.  aux_win_trunk >= 0 is
   * the weight of the win head's gradient into the LSTM ("a very small weight");
   * the rank and building heads are stop_gradient.  All zero = no aux heads. */
  int32_t n_aux_win, n_aux_rank, n_aux_bld;
  float aux_win_trunk;
} ppo_dims;

/* Flat parameter vector theta (fp32 master; grads, Adam m and v share the layout).
 *   W_xh_aug [4H][Kx], Kx = D + H + 64: row r holds gate (r%256)/64 of hidden unit
 *            64*(r/256) + r%64 (gate-interleaved, gates i,f,g,o);
 *            cols [0,D) = W_x, [D,D+H) = W_h, col D+H = LSTM bias b, rest 0.
 *   W_o_aug  [A][Ko],  Ko = H + 64: cols [0,H) = W_o, col H = b_o, rest 0.
 * The zero pad columns receive exactly zero gradient and stay zero under Adam. */
typedef struct {
  int64_t Kx, Ko, A;
  int64_t off_wxh, n_wxh;
  int64_t off_wo, n_wo;
  int64_t n_total;
} ppo_param_layout;

typedef struct {
  float clip_eps; /* PPO clip epsilon, 0.2 */
  float c_v;      /* value loss weight, 1.0 */
  float c_e;      /* entropy coefficient, 0.01 */
  float denom;    /* loss denominator; <= 0 means T*B (DESIGN Q9) */
  float c_win, c_rank, c_bld; /* NEXT-4 aux loss weights (DESIGN Q25); unused without aux */
} ppo_loss_cfg;

/* stats[] layout written by ppo_loss_grad (all Σ_rows w·x / denom unless noted) */
enum {
  PPO_STAT_LOSS = 0, PPO_STAT_PG = 1, PPO_STAT_VF = 2, PPO_STAT_ENT = 3,
  PPO_STAT_KL = 4,        /* approx KL: mean(logp_old - logp) */
  PPO_STAT_CLIPFRAC = 5,  /* rows on the clipped (zero-gradient) side */
  PPO_STAT_NVALID = 6,    /* Σ w */
  PPO_STAT_FLAGS = 7,     /* bit0 non-finite, bit1 taken primary unavailable, bit2 empty avail */
  PPO_STAT_AUX = 8,       /* NEXT-4: the aux part of LOSS, sum of c_k * aux loss k */
  PPO_STATS = 9
};
#define PPO_LOSS_BLOCKS 1184                       /* 148 SMs x 8 */
#define PPO_STATS_BUF (PPO_STATS * (1 + PPO_LOSS_BLOCKS)) /* floats; [0,PPO_STATS) = result */

/* ---- library / errors ---------------------------------------------------------------- */
const char* ppo_last_error(void);                  /* thread-local message of the last error */
const char* ppo_version(void);

/* Host-only: parameter layout for dims (no device access). */
int ppo_get_param_layout(const ppo_dims* dims, ppo_param_layout* out /* host */);

/* Canonical fp32 params (gate blocks [i;f;g;o], PyTorch order, Q14) -> flat theta.
 * Wx [4H][D], Wh [4H][H], b [4H], Wo [A][H], bo [A]; theta [n_total] (fully written). */
int ppo_pack_params(const ppo_dims* dims, const float* Wx, const float* Wh, const float* b,
                    const float* Wo, const float* bo, float* theta, ppo_stream_t s);
/* Inverse of ppo_pack_params (also used to read gradients in canonical layout). */
int ppo_unpack_params(const ppo_dims* dims, const float* theta, float* Wx, float* Wh, float* b,
                      float* Wo, float* bo, ppo_stream_t s);
/* fp32 -> bf16 (round to nearest even) copy of n elements: the tensor-core shadow of theta. */
int ppo_cast_bf16(const float* src, uint16_t* dst, size_t n, ppo_stream_t s);

/* ---- a1: GAE (oracle O2, reading Q10) --------------------------
 * rew [R][L], val [R][L+1] (val[r][L] = bootstrap), done [R][L] (1 = episode ended after
 * step t; zeroes bootstrap and carry).  gamma = 1 - T_step/H_horizon, lam 0.95.
 *   delta_t = r_t + gamma (1-d_t) V_{t+1} - V_t ;  A_t = delta_t + gamma lam (1-d_t) A_{t+1}
 *   R_t = A_t + V_t.
 * seq_T = 0: adv/ret are [R][L].  seq_T = T > 0 (L % T == 0): adv/ret are written time-major
 * for the minibatch, [T][R*L/T], sequence b = r*(L/T) + k covers steps kT..kT+T-1 (O3).
 * fp32 arithmetic.  R*L = 0 is a no-op.
 * L <= 8192 or R >= 600: one warp per stream (L <= 256: per-lane loads; longer streams:
 * windows of 256 steps streamed through TMA bulk copies into a shared-memory ring, 6 windows
 * ahead, when the bases allow it).  Otherwise (few very long rollouts, up to the paper's whole
 * games, ~20k steps, and beyond): chunk-parallel single pass with a decoupled
 * look-back; it needs ppo_gae_scratch_bytes(R, L) bytes of caller-owned, 16-byte aligned
 * device scratch (0 -- scratch may be NULL -- when the warp-per-stream kernels run). */
int ppo_gae_scratch_bytes(int64_t R, int64_t L, size_t* bytes /* host */);
int ppo_gae(const float* rew, const float* val, const uint8_t* done, int64_t R, int64_t L,
            float gamma, float lam, int32_t seq_T, float* adv, float* ret, void* scratch,
            size_t scratch_bytes, ppo_stream_t s);

/* ---- a2-a4: forward (P:1210 LSTM, P:1254 TBPTT-16, P:606/618 heads; O4, O5) ------------
 * Workspace holding the saved activations for lstm_bptt_bwd; caller-owned. */
int lstm_ws_bytes(const ppo_dims* dims, int64_t B, size_t* bytes /* host */);
/* w: weights in the flat theta layout -- the bf16 shadow (uint16) for PPO_PREC_BF16, the fp32
 *    theta itself for PPO_PREC_FP32.
 * x: [T][B][D] LSTM inputs (bf16 bits for BF16, fp32 for FP32); h0, c0: [B][H] fp32 stored
 *    rollout states.  out: [T][B][A] fp32 head outputs (655 logits + value).
 * Computes z_t = [x_t | h_{t-1} | 1] W_xh_aug^T with the cell (i,f,o sigmoid, g tanh,
 * c_t = f c_{t-1} + i g, h_t = o tanh c_t) fused into the GEMM epilogue, then
 * y = [h_t | 1] W_o_aug^T.  1 <= B; ws_bytes >= lstm_ws_bytes().
 * x == NULL: x is already in the workspace -- written by the caller through lstm_ws_x /
 * ppo_copy_x (then h0, c0 are packed as usual) or, with h0 == c0 == NULL too, placed together
 * with h0/c0 by ppo_gather. */
int lstm_bptt_fwd(const ppo_dims* dims, const void* w, const void* x, const float* h0,
                  const float* c0, int64_t B, void* ws, size_t ws_bytes, float* out,
                  ppo_stream_t s);

/* Zero-copy inputs: where x lives inside ws.  Row (t, b) of x starts at *x + (t*B + b) * *ld
 * elements (bf16 for PPO_PREC_BF16, fp32 otherwise); *ld = D + H + 64 >= D.  Rows only carry x
 * in their first D elements; everything else in ws belongs to the library. */
int lstm_ws_x(const ppo_dims* dims, int64_t B, void* ws, void** x /* host out */,
              int64_t* ld /* host out */);
/* Copy x [T*B][D] with row stride src_ld elements (host -- pinned for async -- or device
 * memory) into the workspace rows: one cudaMemcpy2DAsync on the stream. */
int ppo_copy_x(const ppo_dims* dims, int64_t B, const void* src, int64_t src_ld, void* ws,
               size_t ws_bytes, ppo_stream_t s);

/* Streaming inputs: copy time slice t of x (B rows [B][D], row stride src_ld elements; pinned
 * host or device) into the workspace, and run the forward with x already there while the
 * later slices are still in flight: lstm_bptt_fwd_ev waits on x_ready[t] (a cudaEvent_t
 * recorded after slice t's copy; NULL entries or a NULL array = no wait) before step t.
 * h0, c0 as in lstm_bptt_fwd with x == NULL. */
int ppo_copy_x_slice(const ppo_dims* dims, int64_t B, int32_t t, const void* src,
                     int64_t src_ld, void* ws, size_t ws_bytes, ppo_stream_t s);
int lstm_bptt_fwd_ev(const ppo_dims* dims, const void* w, const float* h0, const float* c0,
                     int64_t B, void* ws, size_t ws_bytes, float* out,
                     void* const* x_ready /* host array of T cudaEvent_t */, ppo_stream_t s);

/* ---- a5: PPO loss and its gradient (O6, O7) --
 * out [T·B][A] fp32 (row = t*B + b); act [T·B][n_heads] int32; head_on [T·B][n_heads] u8
 * (heads read by the taken primary action, Table target types P:350-368); avail
 * [T·B][head_sizes[0]] u8 (action filter); logp_old, adv, ret [T·B] fp32;
 * valid [T·B] u8 or NULL (= all rows valid).
 * aux_label [T·B][n_aux] fp32 (n_aux = n_aux_win + n_aux_rank + n_aux_bld; NULL when 0):
 * the NEXT-4 targets from ppo_aux_labels; the aux losses (DESIGN Q25) join the loss.
 * Output columns: [policy logits | value | aux]; the value is column head_off[n_heads].
 * dout [T·B][A]: dL/dout, in the path's activation type (bf16 bits / fp32), consumed by
 * lstm_bptt_bwd; the win column holds aux_win_trunk x its gradient when aux_win_trunk > 0
 * (lstm_bptt_bwd undoes the factor for the win head's own weights, DESIGN Q26).
 * logp [T·B] fp32 or NULL: current log pi(a).  stats [PPO_STATS_BUF]. */
int ppo_loss_grad(const ppo_dims* dims, const float* out, const int32_t* act,
                  const uint8_t* head_on, const uint8_t* avail, const float* logp_old,
                  const float* adv, const float* ret, const uint8_t* valid,
                  const float* aux_label, int64_t B, const ppo_loss_cfg* cfg, void* dout,
                  float* logp, float* stats, ppo_stream_t s);

/* NEXT-4: aux-head targets per 256-step segment (Eq.; DESIGN Q27), computed at
 * ingest like GAE.  R segments of L steps; last [R] u8 (the game's last segment), outcome
 * [R] fp32 (1 = win), rank [R] int32 (0-based final net-worth rank), events [R][L][n_aux_bld]
 * u8 (the hero helped destroy building j at that step), boot [R][n_aux] fp32 (the model's
 * predictions after the segment's last step: win probability, rank distribution, building
 * values), gamma2 = 1 - T_step / 120 s.  labels: seq_T == 0 -> [R][L][n_aux];
 * seq_T > 0 (L % seq_T == 0) -> minibatch layout [seq_T][R*L/seq_T][n_aux] (sequence
 * r*(L/seq_T) + l/seq_T, step l % seq_T), as ppo_gae.  Device pointers; asynchronous. */
int ppo_aux_labels(const ppo_dims* dims, int64_t R, int64_t L, const uint8_t* last,
                   const float* outcome, const int32_t* rank, const uint8_t* events,
                   const float* boot, float gamma2, int32_t seq_T, float* labels,
                   ppo_stream_t s);

/* ---- a6-a8: backward (TBPTT, no gradient into h0/c0; O8) ------------------------
 * ws: the workspace filled by lstm_bptt_fwd for the same (w, B) (it is modified: saved gates
 * are overwritten by dz; with PPO_PREC_BF16 and fewer backward tiles per step than CTA pairs
 * -- small B such as the paper's 600 -- the workspace's split-K region also receives the fp32
 * partials of dh).  dout: from ppo_loss_grad.  grad: [n_total] fp32, OVERWRITTEN with
 * dL/dtheta in the theta layout (bias gradients fall out of the augmented columns).
 * Aux heads (NEXT-4): the LSTM receives the policy, value and (scaled) win columns of dout
 * only; every output row of W_o_aug gets its head's full gradient (DESIGN Q26). */
int lstm_bptt_bwd(const ppo_dims* dims, const void* w, void* ws, size_t ws_bytes,
                  const void* dout, int64_t B, float* grad, ppo_stream_t s);

/* lstm_bptt_bwd that also records wxh_ready (a cudaEvent_t, nullable) on s as soon as the
 * W_xh_aug gradient -- theta [0, off_wo) -- is final, before the W_o gradient GEMM, so the
 * caller can start exchanging it while dW_o computes (ppo_dp_adam_step_range). */
int lstm_bptt_bwd_ev(const ppo_dims* dims, const void* w, void* ws, size_t ws_bytes,
                     const void* dout, int64_t B, float* grad, void* wxh_ready, ppo_stream_t s);

/* NEXT-4: dL/dx for the upstream observation-processing network (the processed
 * observation vector is the LSTM input).  dx[t][b][:] = dz_t[b] W_x for all t, from the dz
 * that lstm_bptt_bwd left in ws (call it after lstm_bptt_bwd, same w, ws, B).
 * dx: [T][B][D] fp32, device, 16-byte aligned, overwritten.  Asynchronous. */
int lstm_input_grad(const ppo_dims* dims, const void* w, const void* ws, size_t ws_bytes,
                    int64_t B, float* dx, ppo_stream_t s);

/* ---- a9: data-parallel gradient average (P:1251 NCCL allreduce; O9) --------------------- */
typedef struct ppo_comm ppo_comm;
#define PPO_COMM_ID_BYTES 128
int ppo_comm_unique_id(uint8_t id[PPO_COMM_ID_BYTES] /* host */);
/* Collective over `world` ranks; call once per rank with the same id (broadcast by the
 * caller, e.g. over a torch process group).  Uses the current CUDA device. */
int ppo_comm_init(const uint8_t id[PPO_COMM_ID_BYTES] /* host */, int rank, int world,
                  ppo_comm** comm /* host out */);
/* In-place average g <- (1/world) sum_ranks g over n fp32 elements, split into n_buckets
 * equal buckets issued in order (n_buckets <= 0 -> 1).  world == 1 is a no-op. */
int grad_allreduce(ppo_comm* comm, float* g, size_t n, int32_t n_buckets, ppo_stream_t s);
int ppo_comm_destroy(ppo_comm* comm);

/* ---- a9+a10 fused over NVLink peer memory (SURVEY §8(e) option: reduce-scatter -> Adam on
 * 1/N of theta -> all-gather; "averaged ... before being synchronously applied").
 * Rank r owns the shard [r s, min(n, (r+1) s)) with s = ppo_dp_shard(n, world).  One kernel
 * per rank reads its shard of every rank's gradient over NVLink (CUDA IPC mappings), sums it
 * in rank order (so the average is the same bits wherever it is formed), scales by 1/world,
 * applies a10 to its shard of theta, m and v, and stores what the forward reads into every
 * rank's copy: the bf16 shadow when there is one (theta, m, v then stay sharded -- current on
 * each rank's own shard only, until ppo_dp_allgather), else theta (fp32 path).  A 1-float
 * NCCL allreduce before and after the kernel orders it against the peers' backward and next
 * forward (stream-ordered; no spinning kernel).  The all-gathered copies are bitwise
 * identical on all ranks. */
#define PPO_DP_MAX_RANKS 8
/* floats per shard (a multiple of 64) */
size_t ppo_dp_shard(size_t n, int world);
/* Collective, synchronous, once per comm: maps every rank's grad g [n] fp32, theta p [n] fp32
 * and shadow p_bf16 [n] bf16 (nullable; the same on every rank) into this process.  The
 * buffers must be cudaMalloc'd device memory (torch's default allocator qualifies; not
 * expandable segments), 16-byte aligned, and stay allocated until ppo_comm_destroy (which
 * closes the mappings).  world == 1: records the pointers only.  Errors are per rank: if any
 * rank's call fails, no rank may use ppo_dp_adam_step on this comm (agree over the caller's
 * process group first, as bench.py does, and fall back to grad_allreduce + adam_step). */
int ppo_dp_attach(ppo_comm* comm, float* g, float* p, uint16_t* p_bf16, size_t n);
/* a9 + a10 for this rank's shard (same arguments and arithmetic as adam_step).  Collective:
 * every rank calls it once per step, after its backward, on the attached buffers.  m, v:
 * [n] fp32, 16-byte aligned; only this rank's shard is read and written.  staged = 0 (pull
 * mode): the shard of every rank's gradient is read over NVLink; staged = 1 (push mode):
 * from this rank's staging, filled by every rank's lstm_bptt_bwd_dp of this step. */
int ppo_dp_adam_step(ppo_comm* comm, float* m, float* v, int64_t t, double lr, double b1,
                     double b2, double eps, double clip_sigma, int32_t staged, ppo_stream_t s);
/* The same exchange restricted to theta elements [lo, hi) (lo a multiple of 64; hi a multiple
 * of 64 or n): each rank updates its shard's part of the range, with the same barriers.  With
 * lstm_bptt_bwd_ev the step overlaps the exchange of W_xh_aug (theta [0, off_wo), 97% of the
 * bytes) with the dW_o GEMM: range [0, off_wo) on a second stream once wxh_ready fires, then
 * [off_wo, n) after the backward.  Every rank must issue the range calls in the same order
 * (they are collective over the comm's NCCL communicator, which serialises them). */
int ppo_dp_adam_step_range(ppo_comm* comm, float* m, float* v, int64_t t, double lr, double b1,
                           double b2, double eps, double clip_sigma, int32_t staged, size_t lo,
                           size_t hi, ppo_stream_t s);
/* Push mode (staged = 1 in ppo_dp_adam_step): the backward itself delivers the gradients --
 * lstm_bptt_bwd, plus: the epilogues of the tiles that produce final weight gradients (the
 * last K-chunk of dW_xh, dW_o's split-K reduction) also store each 4-element group over
 * NVLink into its owner's staging slot for this rank (a library-owned buffer of world x shard
 * floats per rank, mapped by ppo_dp_attach), so the reduce-scatter overlaps the GEMM tile by
 * tile and ppo_dp_adam_step reads only local memory.  Same bits as pull mode.  grad still
 * receives this rank's own gradient (measured: Adam 0.4-0.55 ms instead of 0.75-1.0 ms, but
 * the whole step 1-1.5% slower than pull mode).  bf16 path without the win-head
 * trunk route only (PPO_E_UNSUPPORTED otherwise: use lstm_bptt_bwd + staged = 0); comm
 * attached with world > 1 (PPO_E_ARG otherwise); the attached n must be this model's theta
 * length (PPO_E_SHAPE).  Asynchronous on s, like lstm_bptt_bwd. */
int lstm_bptt_bwd_dp(const ppo_dims* dims, const void* w, void* ws, size_t ws_bytes,
                     const void* dout, int64_t B, float* grad, ppo_comm* comm, ppo_stream_t s);
/* Collective: in-place all-gather of a sharded fp32 vector (m, v, theta before a checkpoint).
 * buf holds world * ppo_dp_shard(n, world) floats (n = the attached length; the slack past n
 * is scratch). */
int ppo_dp_allgather(ppo_comm* comm, float* buf, ppo_stream_t s);

/* Test hook (not part of the step): the fused kernel of ppo_dp_adam_step, run for `world`
 * (1..PPO_DP_MAX_RANKS) VIRTUAL ranks on the current device, so the reduce-scatter / Adam /
 * all-gather arithmetic at world 2, 4 and 8 is checkable on a one-GPU box.  Every argument
 * but n and the scalars is a HOST array of `world` device pointers, entry j = virtual rank
 * j's buffer: g [n] fp32 gradients; p [n] fp32 theta; p_bf16 [n] bf16 shadows (the array, or
 * its entry 0, NULL = fp32 path); m, v [n] fp32 moments; stage (array nullable = pull mode):
 * rank j's push-mode staging of world x ppo_dp_shard(n, world) floats, slot i = rank i's
 * gradient over rank j's shard (what lstm_bptt_bwd_dp delivers).  The kernel is launched once
 * per virtual rank r, in rank order on s, with r's shard [r s, min(n, (r+1) s)); the stream
 * order replaces the two NCCL barriers.  Afterwards, exactly as on `world` GPUs: m[r], v[r]
 * (and p[r] when there is a shadow) are updated on r's shard only; every p_bf16[j] (fp32
 * path: every p[j]) holds the whole updated vector.  16-byte aligned; asynchronous. */
int ppo_test_dp_adam(int32_t world, const float* const* g, float* const* p,
                     uint16_t* const* p_bf16, float* const* m, float* const* v,
                     const float* const* stage, size_t n, int64_t t, double lr, double b1,
                     double b2, double eps, double clip_sigma, ppo_stream_t s);

/* ---- a10: Adam with the +-clip_sigma sqrt(v) clip (O10, Q3, Q4) --
 *   v <- b2 v + (1-b2) g^2;  g_c = clamp(g, +-clip_sigma sqrt(v));  m <- b1 m + (1-b1) g_c
 *   p <- p - lr sqrt(1-b2^t)/(1-b1^t) * m / (sqrt(v) + eps)
 * t >= 1 (step number); clip_sigma <= 0 or inf disables the clip.  p_bf16 (nullable) receives
 * the bf16 shadow of the updated p.  All arrays n fp32 elements (p_bf16: n uint16).
 * Host scalars are double: alpha_t, 1-b1 and 1-b2 are formed in double and rounded once to
 * fp32 (1-b2 from an fp32 b2 would be off by 1.3e-5 relative). */
int adam_step(float* p, uint16_t* p_bf16, const float* g, float* m, float* v, size_t n,
              int64_t t, double lr, double b1, double b2, double eps, double clip_sigma,
              ppo_stream_t s);

/* a10 with the step number on the device, so a captured CUDA graph of the whole step applies
 * the right bias correction on every replay.  ctr: 16 bytes of 16-byte
 * aligned device memory: int64 at byte 0 = steps taken so far (0 before the first step; the
 * call advances it to t), float at byte 8 = scratch (this step's alpha_t).  alpha_t =
 * lr sqrt(1-b2^t)/(1-b1^t) is formed in double on the device and rounded once to fp32 (the
 * same expression as adam_step's host path); otherwise identical to adam_step.  n = 0 is a
 * no-op (the counter does not advance).  Asynchronous; one extra 1-thread launch. */
int adam_step_ctr(float* p, uint16_t* p_bf16, const float* g, float* m, float* v, size_t n,
                  int64_t* ctr, double lr, double b1, double b2, double eps, double clip_sigma,
                  ppo_stream_t s);

/* ---- NEXT-1: experience buffer and minibatch gather ----------
 * The optimizer's experience buffer holds `capacity` sequences (one hero's 16-step sample,
 * P:924) in sequence-major slots, all arrays device memory owned by the caller:
 *   x [cap][T][D] (bf16 bits for PPO_PREC_BF16, fp32 otherwise), h0, c0 [cap][H] fp32,
 *   act [cap][T][n_heads] int32, head_on [cap][T][n_heads] u8, avail [cap][T][head_sizes[0]]
 *   u8, logp_old, adv, ret [cap][T] fp32, valid [cap][T] u8 (NULL = all valid).
 * Rollouts push 256-step segments as 16 consecutive slots; their advantages are
 * computed at ingest with ppo_gae(seq_T = 0) writing adv/ret + slot*T (the segment's 256
 * steps are contiguous there).  Minibatches are sampled uniformly WITH replacement
 * (DESIGN Q19) by a counter-based generator the oracle re-implements:
 *   idx[i] = splitmix64(seed + (step << 32) + i) mod capacity. */
typedef struct {
  const void* x;
  const float *h0, *c0;
  const int32_t* act;
  const uint8_t *head_on, *avail;
  const float *logp_old, *adv, *ret;
  const uint8_t* valid;
  int64_t capacity;
} ppo_buffer;
int ppo_sample_indices(int64_t capacity, int64_t B, uint64_t seed, uint64_t step, int32_t* idx,
                       ppo_stream_t s);
/* Gather B sequences idx[0..B) of the buffer: x, h0, c0 go straight into the workspace (then
 * call lstm_bptt_fwd with x = NULL); the per-timestep loss inputs are written time-major
 * [T][B][.] into act, head_on, avail, logp_old, adv, ret and valid (nullable). */
int ppo_gather(const ppo_dims* dims, const ppo_buffer* buf /* host struct */, const int32_t* idx,
               int64_t B, void* ws, size_t ws_bytes, int32_t* act, uint8_t* head_on,
               uint8_t* avail, float* logp_old, float* adv, float* ret, uint8_t* valid,
               ppo_stream_t s);

/* ---- NEXT-2: reward pipeline fused into GAE (App. Reward Weights P:1058-1079) -----
 * Per game g and hero i (0-4 one team, 5-9 the other; stream s = 10 g + i):
 *   rho_i = shaped_i * decay_base^(t_game / decay_seconds) + win_i,   t_game = (step0[g] + l)
 *           * step_seconds   (0.6^(T / 10 min); win/loss exempt)
 *   r_i   = (1 - tau) rho_i + tau mean_team(rho) - [zero_sum] mean_enemy(rho)
 *   r_i  /= sigma, the running std of all final rewards of PREVIOUS calls (1 before any data);
 *           this call's r then updates stats = {count, mean, M2} (device, fp64)
 *   then GAE exactly as ppo_gae on the normalised rewards (streams of length L, seq_T layout).
 * shaped, win [G][10][L]; step0 [G] int32; val [10G][L+1]; done [G][L] (per game); adv, ret
 * and rew_out (nullable: normalised r) laid out like ppo_gae's outputs for R = 10 G.
 * scratch: ppo_reward_gae_scratch_bytes() of 8-byte aligned device memory.  DESIGN Q20, Q21. */
typedef struct {
  float tau;            /* team spirit, 0.3 -> 0.8 in Rerun */
  float decay_base;     /* 0.6 */
  float decay_seconds;  /* 600 (10 minutes of game time) */
  float step_seconds;   /* 4/30 (frameskip 4 at 30 fps) */
  int32_t zero_sum;     /* 1: subtract the enemy team's mean reward */
} ppo_reward_cfg;
int ppo_reward_gae_scratch_bytes(size_t* bytes /* host */);
int ppo_reward_gae(const float* shaped, const float* win, const int32_t* step0, int64_t G,
                   int64_t L, const float* val, const uint8_t* done, const ppo_reward_cfg* cfg,
                   double* stats, float gamma, float lam, int32_t seq_T, float* rew_out,
                   float* adv, float* ret, void* scratch, size_t scratch_bytes, ppo_stream_t s);

/* ---- NEXT-3: forward-pass inference step ---------------------------------------
 * "a separate pool of GPU machines which run forward passes in larger batches of
 * approximately 60": one policy step for B heroes.
 *   z = W_xh_aug [x | h | 1]; LSTM cell -> h', c' (written back in place);
 *   x is read by TMA directly from the caller's buffer (rows of D*2 bytes, 16-byte aligned)
 *   y = W_o_aug [h' | 1]  (logits of the n_heads heads | value)
 *   act[b][k] = argmax over allowed j of (y_kj + g_kj), g = -log(-log u) Gumbel noise, ties
 *     to the smallest j (DESIGN reading Q22); allowed = avail[b] for the primary head (action
 *     filters), every entry for the parameter heads;
 *     u(b, j) = ((splitmix64(seed + (step << 32) + 1024 b + j) >> 41) + 1/2) / 2^23 over the
 *     concatenated head logits j (the oracle implements the same counter generator);
 *   head_on[b] = head_table[act[b][0]] (Table target types);
 *   logp[b] = sum_k head_on[b][k] log softmax_allowed(y_k)[act[b][k]] (behaviour log-prob);
 *   value[b] = y[b][A-1].
 * A row with no available primary (reading Q23) gets act[b][0] = -1, head_on 0, logp 0.
 * Layouts: w = weights tiled by ppo_infer_pack_weights; x [B][D] bf16 bits; h, c [B][H] fp32,
 * updated in place; avail [B][head_sizes[0]] uint8; head_table [head_sizes[0]][n_heads]
 * uint8; act [B][n_heads] int32; head_on [B][n_heads] uint8 (may be NULL); logp [B] fp32;
 * value [B] (may be NULL); out [B][A] fp32 head outputs (may be NULL).  All device
 * pointers; w, x, h, c 16-byte aligned; ws 1024-byte aligned, >= ppo_infer_ws_bytes.
 * bf16 precision only (PPO_E_ARG otherwise); PPO_E_UNSUPPORTED off sm_100.
 * Asynchronous on the stream. */
/* Same step with the counter on the device: this call draws with step = *step_ctr and leaves
 * *step_ctr + 1 (device uint64, 8-byte aligned), so a captured CUDA graph of inference steps
 * draws fresh noise on every replay.  flags: PPO_INFER_STATE_CURRENT = the workspace still
 * holds the bf16 copy of h written by this ws's previous step (h not modified since): the
 * state upload is skipped.  Without it (first call, or after the caller changed h) the step
 * re-derives the copy from h. */
#define PPO_INFER_STATE_CURRENT 1u
int ppo_infer_step_ctr(const ppo_dims* dims, const void* w, const void* x, float* h, float* c,
                       const uint8_t* avail, const uint8_t* head_table, uint64_t seed,
                       uint64_t* step_ctr, uint32_t flags, int64_t B, void* ws,
                       size_t ws_bytes, int32_t* act, uint8_t* head_on, float* logp,
                       float* value, float* out, ppo_stream_t s);
int ppo_infer_ws_bytes(const ppo_dims* dims, int64_t B, size_t* bytes /* host out */);
/* The served weights, re-laid out once per published version for streaming: every
 * [128 rows][64 k] block of W_xh_aug and W_o_aug becomes one contiguous 16 KB tile (rows past
 * the matrix zero), gates then heads.  w: the bf16 shadow in ppo_param_layout (device);
 * wt: device, 16-byte aligned, >= ppo_infer_weights_bytes. */
int ppo_infer_weights_bytes(const ppo_dims* dims, size_t* bytes /* host out */);
int ppo_infer_pack_weights(const ppo_dims* dims, const void* w, void* wt, size_t wt_bytes,
                           ppo_stream_t s);
int ppo_infer_step(const ppo_dims* dims, const void* w, const void* x, float* h, float* c,
                   const uint8_t* avail, const uint8_t* head_table, uint64_t seed,
                   uint64_t step, int64_t B, void* ws, size_t ws_bytes, int32_t* act,
                   uint8_t* head_on, float* logp, float* value, float* out, ppo_stream_t s);

/* ---- device topology (diagnostics) ---------------------------------------------------------
 * SMs of the current device and how they split over its dies (B200: two dies; an address is
 * homed on one of them, and the CTA-pair GEMMs give each die its own tile queue so the tiles
 * sharing operand panels run on one die).  Measured once per device by a latency probe
 * (~1 ms, on first use); *die0 = *die1 = 0 when no two-die split was found (then one queue).
 * Synchronous; not callable during stream capture (returns the cached result or zeros). */
int ppo_device_info(int32_t* n_sms /* host */, int32_t* die0_sms /* host */,
                    int32_t* die1_sms /* host */);

/* ---- tracing: CUDA events around every kernel launch ------------------------
 * ppo_prof_start() enables recording (clears previous records); every library launch then
 * records a start/end event pair on its stream.  ppo_prof_stop() synchronises those events,
 * aggregates per kernel tag (launch count, total device ms, in first-seen order) into
 * out[0..max_entries) (host), sets *n_out to the number of tags and disables recording. */
typedef struct {
  char name[32];
  int32_t launches;
  double total_ms;
} ppo_prof_entry;
int ppo_prof_start(void);
int ppo_prof_stop(ppo_prof_entry* out /* host */, int32_t max_entries, int32_t* n_out /* host */);

/* ---- testing hook (not part of the step) -------------------------------------------------
 * One standalone tcgen05 GEMM C[M][N] (fp32) = sum_k A(m,k) B(n,k) on bf16 operands, used by
 * the kernel unit tests.  mode bit0: B stored MN-major [K][N] (else K-major [N][K]);
 * bit1: A stored MN-major [K][M] (else [M][K]); bit2: N-tile 224 instead of 256. */
int ppo_test_tc_gemm(int mode, const uint16_t* A, const uint16_t* B, float* C, int M, int N,
                     int K, ppo_stream_t s);

#ifdef __cplusplus
}
#endif
#endif /* PPO5_H */
