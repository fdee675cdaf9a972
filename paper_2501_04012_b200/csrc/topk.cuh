// topk.cuh — block-level exact top-k selection by (score desc, id asc).
//
// Used by the exact scan, the fp64 rescore and the shard merge. The order is
// the generalisation of query_top1's strict '>' over ascending ids
// (vindex.cpp:58-72): for k = 1 it returns exactly the reference's answer.
#pragma once
#include "common.cuh"

namespace fc {

struct Cand {
  double s;
  uint64_t id;
  int64_t slot;  // table row (or -1)
};

__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) { return better(a.s, a.id, b.s, b.id); }

// Sorted insertion into a per-thread list of length <= K (descending).
template <int KMAX>
__device__ __forceinline__ void local_insert(Cand (&L)[KMAX], int& n, int k, const Cand& c) {
  if (n == k && !cand_better(c, L[k - 1])) return;
  int pos = n < k ? n : k - 1;
  while (pos > 0 && cand_better(c, L[pos - 1])) {
    L[pos] = L[pos - 1];
    --pos;
  }
  L[pos] = c;
  if (n < k) ++n;
}

__device__ __forceinline__ void warp_argbest(Cand& c, int& owner) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    Cand o;
    o.s = __shfl_xor_sync(0xffffffffu, c.s, off);
    o.id = __shfl_xor_sync(0xffffffffu, c.id, off);
    o.slot = __shfl_xor_sync(0xffffffffu, c.slot, off);
    int oo = __shfl_xor_sync(0xffffffffu, owner, off);
    // tie on (s, id) impossible for distinct items; owner breaks exact dups
    if (oo >= 0 && (owner < 0 || cand_better(o, c) || (!cand_better(c, o) && oo < owner))) {
      c = o;
      owner = oo;
    }
  }
}

// Each thread contributes a descending list L[0..n). The block extracts the
// global top-k (k rounds of a block-wide argmax over list heads) into
// out[0..k) and returns the count (thread 0's value is authoritative; all
// threads return it). smem: needs (blockDim/32) Cand + int scratch.
template <int KMAX>
__device__ int block_merge_lists(Cand (&L)[KMAX], int n, int k, Cand* out, Cand* s_c, int* s_o) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int ptr = 0;
  int produced = 0;
  __shared__ int s_total;
  for (int r = 0; r < k; ++r) {
    Cand c;
    int owner;
    if (ptr < n) {
      c = L[ptr];
      owner = threadIdx.x;
    } else {
      c.s = 0; c.id = 0; c.slot = -1;
      owner = -1;
    }
    warp_argbest(c, owner);
    if (lane == 0) {
      s_c[warp] = c;
      s_o[warp] = owner;
    }
    __syncthreads();
    if (warp == 0) {
      Cand d;
      int o2;
      if (lane < nw) {
        d = s_c[lane];
        o2 = s_o[lane];
      } else {
        d.s = 0; d.id = 0; d.slot = -1;
        o2 = -1;
      }
      warp_argbest(d, o2);
      if (lane == 0) {
        s_o[0] = o2;
        s_c[0] = d;
      }
    }
    __syncthreads();
    const int win = s_o[0];
    if (win < 0) break;
    if (threadIdx.x == 0) out[r] = s_c[0];
    if (threadIdx.x == win) ++ptr;
    ++produced;
    __syncthreads();
  }
  if (threadIdx.x == 0) s_total = produced;
  __syncthreads();
  return s_total;
}

}  // namespace fc
