// K8: dataset-sharded top-k merge.  The reference has no sharding; the merge
// order is the one merge_team_results uses (engine.cpp:24-34): ascending
// (dist, id), ids deduplicated, first k.  Each shard's list is already sorted
// by (dist, local id); adding the shard's constant id offset keeps it sorted,
// so one thread per query runs a G-way merge.
#include "common.cuh"
#include "kernels.hpp"

namespace cagra {
namespace {

constexpr int MAX_SHARDS = 64;

__global__ void shard_merge_kernel(const uint32_t* __restrict__ sids,
                                   const float* __restrict__ sdists, uint32_t G, uint32_t nq,
                                   uint32_t k, const uint64_t* __restrict__ offsets,
                                   uint32_t* __restrict__ out_ids,
                                   float* __restrict__ out_dists) {
  uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  uint32_t pos[MAX_SHARDS];
  for (uint32_t g = 0; g < G; ++g) pos[g] = 0;
  uint32_t w = 0, prev = kInvalidId;
  while (w < k) {
    int best = -1;
    uint64_t bkey = 0;
    for (uint32_t g = 0; g < G; ++g) {
      if (pos[g] >= k) continue;
      size_t at = ((size_t)g * nq + q) * k + pos[g];
      uint32_t lid = sids[at];
      if (lid == kInvalidId) continue;
      uint64_t key = make_key(sdists[at], (uint32_t)(lid + offsets[g]));
      if (best < 0 || key < bkey) {
        best = (int)g;
        bkey = key;
      }
    }
    if (best < 0) break;
    pos[best]++;
    uint32_t id = key_id(bkey);
    if (id == prev) continue;
    prev = id;
    out_ids[(size_t)q * k + w] = id;
    out_dists[(size_t)q * k + w] = key_dist(bkey);
    ++w;
  }
  for (; w < k; ++w) {
    out_ids[(size_t)q * k + w] = kInvalidId;
    out_dists[(size_t)q * k + w] = __uint_as_float(0x7f800000u);
  }
}

}  // namespace

void launch_shard_merge(const uint32_t* d_shard_ids, const float* d_shard_dists,
                        uint32_t shards, uint32_t nq, uint32_t k, const uint64_t* d_offsets,
                        uint32_t* d_ids, float* d_dists, cudaStream_t stream) {
  if (shards > MAX_SHARDS) throw UsageErr("shard merge supports at most 64 shards");
  if (nq == 0) return;
  shard_merge_kernel<<<(nq + 127) / 128, 128, 0, stream>>>(d_shard_ids, d_shard_dists, shards, nq,
                                                         k, d_offsets, d_ids, d_dists);
  CAGRA_LAUNCH_CHECK();
}

}  // namespace cagra
