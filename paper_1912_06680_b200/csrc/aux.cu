// aux.cu -- NEXT-4: targets of the auxiliary prediction heads (Eq.; DESIGN Q27),
// computed per 256-step segment at ingest, in the minibatch layout the loss kernel reads.
//   win      y = outcome on the game's last segment, else the model's prediction y_hat(t2)
//   rank     y = onehot(final rank) on the last segment, else the predicted distribution
//   building y_t = 1 if the event happens at step t else gamma2 * y_{t+1};
//            y_L = 0 on the last segment (the game is over) else y_hat_j   (2-min discount)
#include "kernels.cuh"

namespace ppo {
namespace {

__device__ __forceinline__ int64_t label_index(int64_t r, int64_t l, int c, int64_t R, int64_t L,
                                               int seq_T, int n_aux) {
  if (seq_T <= 0) return (r * L + l) * n_aux + c;
  const int64_t per = L / seq_T;                 // sequences per segment
  const int64_t b = r * per + l / seq_T, t = l % seq_T;
  return (t * (R * per) + b) * n_aux + c;
}

// One thread per (segment r, label column c).
__global__ void aux_labels_kernel(int64_t R, int64_t L, int n_win, int n_rank, int n_bld,
                                  const uint8_t* __restrict__ last,
                                  const float* __restrict__ outcome,
                                  const int32_t* __restrict__ rank,
                                  const uint8_t* __restrict__ events,
                                  const float* __restrict__ boot, float gamma2, int seq_T,
                                  float* __restrict__ labels) {
  const int n_aux = n_win + n_rank + n_bld;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= R * n_aux) return;
  const int64_t r = e / n_aux;
  const int c = (int)(e - r * n_aux);
  const bool is_last = last[r] != 0;
  if (c < n_win + n_rank) {
    float y;
    if (c < n_win) y = is_last ? outcome[r] : boot[r * n_aux + c];
    else y = is_last ? (rank[r] == c - n_win ? 1.f : 0.f) : boot[r * n_aux + c];
    for (int64_t l = 0; l < L; ++l) labels[label_index(r, l, c, R, L, seq_T, n_aux)] = y;
  } else {
    const int j = c - n_win - n_rank;
    float y = is_last ? 0.f : boot[r * n_aux + c];
    for (int64_t l = L - 1; l >= 0; --l) {
      y = events[(r * L + l) * n_bld + j] ? 1.f : gamma2 * y;
      labels[label_index(r, l, c, R, L, seq_T, n_aux)] = y;
    }
  }
}

}  // namespace
}  // namespace ppo

using namespace ppo;

extern "C" int ppo_aux_labels(const ppo_dims* dims, int64_t R, int64_t L, const uint8_t* last,
                              const float* outcome, const int32_t* rank, const uint8_t* events,
                              const float* boot, float gamma2, int32_t seq_T, float* labels,
                              ppo_stream_t st_) {
  cudaStream_t st = (cudaStream_t)st_;
  Shape s;
  int rc = check_dims(dims, &s);
  if (rc) return rc;
  if (s.n_aux == 0) return PPO_OK;
  if (R < 1 || L < 1) return fail(PPO_E_SHAPE, "R and L must be >= 1");
  if (seq_T > 0 && L % seq_T) return fail(PPO_E_SHAPE, "L must be a multiple of seq_T");
  if (!last || !boot || !labels || (s.n_win && !outcome) || (s.n_rank && !rank) ||
      (s.n_bld && !events))
    return fail(PPO_E_ARG, "NULL pointer");
  if (!(gamma2 >= 0.f && gamma2 <= 1.f)) return fail(PPO_E_ARG, "gamma2 must be in [0, 1]");
  ProfScope _prof("aux_labels", st);
  const int64_t n = R * s.n_aux;
  aux_labels_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(
      R, L, s.n_win, s.n_rank, s.n_bld, last, outcome, rank, events, boot, gamma2, seq_T, labels);
  PPO_LAUNCH_CHECK("aux_labels_kernel");
  return PPO_OK;
}
