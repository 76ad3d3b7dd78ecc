// comm.cu -- a9: data-parallel gradient average ("Gradients are averaged across the
// pool using NCCL2 allreduce before being synchronously applied").  libppo5 owns its NCCL
// communicator; the unique id travels over the caller's torch process group.
#include <nccl.h>

#include <string>

#include "common.cuh"

struct ppo_comm {
  ncclComm_t comm;
  int rank, world;
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
  ncclResult_t r = ncclCommDestroy(c->comm);
  delete c;
  if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
  return PPO_OK;
}

}  // extern "C"
