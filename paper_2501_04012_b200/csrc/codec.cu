// codec.cu — latent codec (codec.hpp:69-118) + stitch (stitcher.cpp:7-39).
//
// Compress pipeline for a batch of n prompts x S steps x F frames x E floats
// (all device-resident):
//   K5 k_gram     F x F Gram matrix per (prompt, step): sequential fp64 dot
//                 products over E (== frame_similarity's sums, core.cpp:101-114),
//                 8x8 register-blocked, frames staged through smem as fp64.
//   K6 k_select   forward greedy key-frame selection (codec.cpp:138-165)
//                 from the Gram matrix; one thread per (prompt, step).
//   K7 k_inter    per (prompt, common key m): differentials, least-squares
//                 alphas (codec.cpp:181-191) for every (step, base) pair,
//                 reconstructs_exactly (codec.cpp:41-46) and the trial
//                 reconstruction similarities (codec.cpp:243-259).
//   host          base selection (strict '>' over ascending steps on the mean
//                 trial similarity) and entry assembly (codec.cpp:52-108) on
//                 the small per-key results.
//   K8 k_pack     frame/mask/recipe copies into the per-entry HBM layout.
// Every fp64 reduction keeps the reference's element order, so maps, base
// step, alphas, extra sets and wire bytes are bit-identical to the reference.
//
// Decompress (K9) is a pure streaming kernel over precomputed per-frame
// recipes; the decoupled-hit variant fuses the mask select of stitch() so
// each output pixel is reconstructed only from the source it is taken from.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "entry.hpp"

namespace fc {

EntryData::~EntryData() {
  if (dev) {
    DeviceGuard g(ctx->device);
    cudaFreeAsync(dev, ctx->stream);
  }
}

lc_entry* make_entry_view(const std::shared_ptr<EntryData>& d, std::vector<int> sel) {
  auto* e = new lc_entry();
  e->d = d;
  e->sel = std::move(sel);
  return e;
}

uint64_t entry_compressed_size(const lc_entry* e) {
  uint64_t n = e->d->shared_bytes();
  for (int si : e->sel) n += e->d->private_bytes(si);
  return n;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
__global__ void k_nonfinite(const float* __restrict__ v, int64_t n, int* __restrict__ bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(v[i])) {
      atomicExch(bad, 1);
      return;
    }
}

// Gram matrix per (prompt, step) item. Thread = one 8x8 block (bj >= bk) of
// frame pairs with 64 fp64 accumulators; chunk = CH elements of every frame.
constexpr int GRAM_SMEM = 32 * 1024 + 2 * 8 * 32 * 16;
__global__ void __launch_bounds__(64) k_gram(const float* __restrict__ lat, int F, int64_t E, double* __restrict__ G) {
  extern __shared__ double s_x[];  // [CH][FP + 2]
  const int FP = (F + 7) & ~7;
  const int NB = FP / 8;
  const int CH = 4096 / FP;
  const int LD = FP + 2;
  const int item = blockIdx.x;
  const float* X = lat + (int64_t)item * F * E;
  const int NP = NB * (NB + 1) / 2;
  int bj = 0, bk = 0;
  {
    int t = threadIdx.x, r = 0;
    while (r < NB && t > r) {
      t -= r + 1;
      ++r;
    }
    bj = r;
    bk = t;
  }
  const bool active = threadIdx.x < NP;
  double acc[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) acc[a][b] = 0.0;
  for (int64_t c0 = 0; c0 < E; c0 += CH) {
    const int cn = (int)min((int64_t)CH, E - c0);
    __syncthreads();
    for (int idx = threadIdx.x; idx < FP * CH; idx += blockDim.x) {
      const int f = idx / CH, i = idx - f * CH;
      s_x[i * LD + f] = (f < F && i < cn) ? (double)X[(int64_t)f * E + c0 + i] : 0.0;
    }
    __syncthreads();
    if (active) {
      for (int i = 0; i < cn; ++i) {
        const double* row = s_x + i * LD;
        double xj[8], xk[8];
#pragma unroll
        for (int a = 0; a < 8; ++a) {
          xj[a] = row[bj * 8 + a];
          xk[a] = row[bk * 8 + a];
        }
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 8; ++b) acc[a][b] = fma(xj[a], xk[b], acc[a][b]);
      }
    }
  }
  if (!active) return;
  double* g = G + (int64_t)item * F * F;
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      const int j = bj * 8 + a, k = bk * 8 + b;
      if (j < F && k < F) {
        g[(int64_t)j * F + k] = acc[a][b];
        g[(int64_t)k * F + j] = acc[a][b];
      }
    }
}

// Greedy forward key-frame selection (codec.cpp:146-163) on the Gram matrix:
// sim(j,k) = G[j][k] / (sqrt(G[j][j]) * sqrt(G[k][k])) (core.cpp:113).
__global__ void k_select(const double* __restrict__ G, int n_items, int F, double thr, int32_t* __restrict__ maps,
                         int* __restrict__ bad) {
  const int item = blockIdx.x * blockDim.x + threadIdx.x;
  if (item >= n_items) return;
  const double* g = G + (int64_t)item * F * F;
  int32_t* map = maps + (int64_t)item * F;
  int keys[256];
  int nk = 0;
  map[0] = 0;
  keys[nk++] = 0;
  if (F >= 2) {
    for (int j = 0; j < F; ++j)
      if (g[(int64_t)j * F + j] == 0.0) {  // cosine_similarity throws (core.cpp:111-112)
        atomicExch(bad, 1);
        return;
      }
  }
  for (int j = 1; j < F; ++j) {
    int best = -1;
    double best_sim = 0.0;
    const double sj = sqrt(g[(int64_t)j * F + j]);
    for (int t = 0; t < nk; ++t) {
      const int k = keys[t];
      const double sim = g[(int64_t)j * F + k] / (sj * sqrt(g[(int64_t)k * F + k]));
      if (sim >= thr && (best < 0 || sim > best_sim)) {
        best = k;
        best_sim = sim;
      }
    }
    if (best < 0) {
      map[j] = j;
      keys[nk++] = j;
    } else {
      map[j] = best;
    }
  }
}

__global__ void k_diag(const double* __restrict__ G, int64_t n_items, int F, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n_items * F) return;
  const int64_t item = i / F, j = i - item * F;
  out[i] = G[item * F * F + j * F + j];
}

constexpr int MAXS = 8;
struct InterRes {
  double sim[MAXS][MAXS];    // [s][b]: safe_similarity(recon_s under base b, key_s)
  float alpha[MAXS][MAXS];   // [s][b]
  uint8_t nz[MAXS];          // diff_s[m] not all zero
  uint8_t exact[MAXS];       // first_s + diff_s == key_s (codec.cpp:41-46)
  uint8_t nonfinite[MAXS][MAXS];
};

struct InterItem {
  int32_t entry;
  int32_t m;
};

// One block per (prompt, common key m > 0). Steps are in ascending order
// through perm (sorted index -> input index).
constexpr int INTER_T = 64;
constexpr int INTER_CH = 256;
__global__ void __launch_bounds__(INTER_T) k_inter(const float* __restrict__ lat, const InterItem* __restrict__ items,
                                                   int S, const int* __restrict__ perm, int F, int64_t E,
                                                   const double* __restrict__ G, InterRes* __restrict__ out) {
  __shared__ float s_key[MAXS][INTER_CH];
  __shared__ float s_first[MAXS][INTER_CH];
  __shared__ double s_num[MAXS][MAXS];
  __shared__ float s_alpha[MAXS][MAXS];
  __shared__ int s_nz[MAXS], s_exact[MAXS];
  const InterItem it = items[blockIdx.x];
  const int m = it.m;
  const float* base = lat + (int64_t)it.entry * S * F * E;
  const int tid = threadIdx.x;
  const int s = tid / MAXS, b = tid % MAXS;  // (s, b) pair of this thread
  const bool pa = s < S && b < S;
  double acc = 0.0;
  bool nz = false, exact = true;
  // ---- phase A: num[s][b] = sum d_s * d_b (den = num[b][b]) ----
  for (int64_t c0 = 0; c0 < E; c0 += INTER_CH) {
    const int cn = (int)min((int64_t)INTER_CH, E - c0);
    __syncthreads();
    for (int idx = tid; idx < S * INTER_CH; idx += INTER_T) {
      const int ss = idx / INTER_CH, i = idx - ss * INTER_CH;
      if (i < cn) {
        const float* st = base + (int64_t)perm[ss] * F * E;
        s_key[ss][i] = st[(int64_t)m * E + c0 + i];
        s_first[ss][i] = st[c0 + i];
      }
    }
    __syncthreads();
    if (pa) {
      for (int i = 0; i < cn; ++i) {
        const float ds = s_key[s][i] - s_first[s][i];
        const float db = s_key[b][i] - s_first[b][i];
        acc = fma((double)ds, (double)db, acc);
        if (s == b) {
          nz |= ds != 0.0f;
          exact &= (s_first[s][i] + ds) == s_key[s][i];
        }
      }
    }
  }
  if (pa) s_num[s][b] = acc;
  if (pa && s == b) {
    s_nz[s] = nz;
    s_exact[s] = exact;
  }
  __syncthreads();
  if (pa) {
    float a = 0.0f;
    if (s_nz[b]) a = (float)(s_num[s][b] / s_num[b][b]);
    s_alpha[s][b] = a;
  }
  __syncthreads();
  // ---- phase B: trial reconstruction of key m of step s under base b ----
  const bool pb = pa && s != b && s_nz[b] && isfinite(s_alpha[s][b]);
  const double alpha = pa ? (double)s_alpha[s][b] : 0.0;
  double dot = 0.0, na = 0.0;
  bool nonfin = false;
  for (int64_t c0 = 0; c0 < E; c0 += INTER_CH) {
    const int cn = (int)min((int64_t)INTER_CH, E - c0);
    __syncthreads();
    for (int idx = tid; idx < S * INTER_CH; idx += INTER_T) {
      const int ss = idx / INTER_CH, i = idx - ss * INTER_CH;
      if (i < cn) {
        const float* st = base + (int64_t)perm[ss] * F * E;
        s_key[ss][i] = st[(int64_t)m * E + c0 + i];
        s_first[ss][i] = st[c0 + i];
      }
    }
    __syncthreads();
    if (pb) {
      for (int i = 0; i < cn; ++i) {
        const float db = s_key[b][i] - s_first[b][i];
        const float r = (float)fma(alpha, (double)db, (double)s_first[s][i]);
        nonfin |= !isfinite(r);
        dot = fma((double)r, (double)s_key[s][i], dot);
        na = fma((double)r, (double)r, na);
      }
    }
  }
  InterRes* o = out + blockIdx.x;
  if (pa) {
    o->alpha[s][b] = s_alpha[s][b];
    o->nonfinite[s][b] = nonfin;
    double sim = 0.0;
    if (pb) {
      const double nb = G[((int64_t)it.entry * S + perm[s]) * F * F + (int64_t)m * F + m];
      if (na == 0.0 && nb == 0.0) sim = 1.0;
      else if (na == 0.0 || nb == 0.0) sim = 0.0;
      else sim = dot / (sqrt(na) * sqrt(nb));
    }
    o->sim[s][b] = sim;
    if (s == b) {
      o->nz[s] = s_nz[s];
      o->exact[s] = s_exact[s];
    }
  }
}

struct FrameJob {
  float* dst;
  const float* src;
  const float* sub;  // dst = src - sub (diff) when non-null
};
struct ByteJob {
  uint8_t* dst;
  const uint8_t* src;
  int64_t n;
};

__global__ void k_pack_frames(const FrameJob* __restrict__ jobs, int64_t E) {
  const FrameJob j = jobs[blockIdx.y];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x)
    j.dst[i] = j.sub ? j.src[i] - j.sub[i] : j.src[i];
}

__global__ void k_pack_bytes(const ByteJob* __restrict__ jobs) {
  const ByteJob j = jobs[blockIdx.y];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < j.n; i += (int64_t)gridDim.x * blockDim.x)
    j.dst[i] = j.src[i];
}

// ---- decompress / stitch ----
struct DecItem {
  const float* base;
  const Recipe* rec;  // [F]
  float* out;         // [F][E]
};

__device__ __forceinline__ float recon(const float* base, const Recipe& r, int64_t i) {
  const float a = base[r.a + i];
  if (r.kind == 0) return a;
  const float b = base[r.b + i];
  if (r.kind == 1) return a + b;
  return (float)fma((double)r.alpha, (double)b, (double)a);
}

__device__ __forceinline__ float4 recon4(const float* base, const Recipe& r, int64_t i) {
  const float4 a = *reinterpret_cast<const float4*>(base + r.a + i);
  if (r.kind == 0) return a;
  const float4 b = *reinterpret_cast<const float4*>(base + r.b + i);
  if (r.kind == 1) return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
  const double al = r.alpha;
  return make_float4((float)fma(al, (double)b.x, (double)a.x), (float)fma(al, (double)b.y, (double)a.y),
                     (float)fma(al, (double)b.z, (double)a.z), (float)fma(al, (double)b.w, (double)a.w));
}

// One block per output frame (grid.x = item * F + frame): the recipe is
// block-uniform, so the kind branch is hoisted out of the streaming loop and
// each thread keeps DEC_U float4 loads (x2 for two-source kinds) in flight.
// Loads use the read-only path; stores are streaming (.cs): the output is
// written once and not re-read by this kernel.
constexpr int DEC_T = 256, DEC_U = 4;
template <int KIND>
__device__ __forceinline__ void dec_frame(const float* __restrict__ a, const float* __restrict__ b, float alpha,
                                          float* __restrict__ out, int64_t n4) {
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  float4* o4 = reinterpret_cast<float4*>(out);
  const double al = alpha;
  for (int64_t i0 = threadIdx.x; i0 < n4; i0 += (int64_t)DEC_T * DEC_U) {
    float4 va[DEC_U], vb[DEC_U];
#pragma unroll
    for (int u = 0; u < DEC_U; ++u) {
      const int64_t i = i0 + (int64_t)u * DEC_T;
      if (i < n4) {
        va[u] = __ldg(a4 + i);
        if (KIND != 0) vb[u] = __ldg(b4 + i);
      }
    }
#pragma unroll
    for (int u = 0; u < DEC_U; ++u) {
      const int64_t i = i0 + (int64_t)u * DEC_T;
      if (i >= n4) break;
      float4 r = va[u];
      if (KIND == 1) {
        r = make_float4(va[u].x + vb[u].x, va[u].y + vb[u].y, va[u].z + vb[u].z, va[u].w + vb[u].w);
      } else if (KIND == 2) {
        r = make_float4((float)fma(al, (double)vb[u].x, (double)va[u].x), (float)fma(al, (double)vb[u].y, (double)va[u].y),
                        (float)fma(al, (double)vb[u].z, (double)va[u].z), (float)fma(al, (double)vb[u].w, (double)va[u].w));
      }
      __stcs(o4 + i, r);
    }
  }
}

__global__ void __launch_bounds__(DEC_T) k_decompress(const DecItem* __restrict__ items, int F, int64_t E) {
  const int item = blockIdx.x / F, j = blockIdx.x - item * F;
  const DecItem it = items[item];
  const Recipe r = it.rec[j];
  float* out = it.out + (int64_t)j * E;
  if ((E & 3) == 0) {
    const int64_t n4 = E >> 2;
    const float* a = it.base + r.a;
    const float* b = it.base + r.b;
    if (r.kind == 0) dec_frame<0>(a, b, r.alpha, out, n4);
    else if (r.kind == 1) dec_frame<1>(a, b, r.alpha, out, n4);
    else dec_frame<2>(a, b, r.alpha, out, n4);
  } else {
    for (int64_t x = threadIdx.x; x < E; x += DEC_T) out[x] = recon(it.base, r, x);
  }
}

struct StitchItem {
  const float* obase;
  const Recipe* orec;
  const float* bbase;
  const Recipe* brec;
  const uint8_t* om;  // object-source object masks [F][mb]
  const uint8_t* sm;  // background-source object masks [F][mb]
  float* out;
};

__device__ __forceinline__ bool mask_bit(const uint8_t* m, int64_t p) { return (m[p >> 3] >> (p & 7)) & 1; }

// Fused decompress(obj) / decompress(bg) / stitch: pixel p of frame j is the
// object source's iff objsrc.object_mask | bgsrc.object_mask (stitcher.cpp:25-37).
// One block per output frame; the frame's two mask planes are OR-ed into
// shared memory once, then each float4 (one pixel when C == 4) reads only the
// source its bit selects.
__global__ void __launch_bounds__(DEC_T) k_decompress_stitch(const StitchItem* __restrict__ items, int F, int64_t E,
                                                             int C, int64_t mb) {
  extern __shared__ uint8_t s_m[];  // [mb] OR of the two object masks
  const int item = blockIdx.x / F, j = blockIdx.x - item * F;
  const StitchItem it = items[item];
  const Recipe ro = it.orec[j], rb = it.brec[j];
  const uint8_t* om = it.om + (int64_t)j * mb;
  const uint8_t* sm = it.sm + (int64_t)j * mb;
  for (int64_t x = threadIdx.x; x < mb; x += DEC_T) s_m[x] = om[x] | sm[x];
  __syncthreads();
  float* out = it.out + (int64_t)j * E;
  if (C == 4) {
    float4* o4 = reinterpret_cast<float4*>(out);
    const int64_t n4 = E >> 2;
    for (int64_t i0 = threadIdx.x; i0 < n4; i0 += (int64_t)DEC_T * DEC_U) {
      float4 r[DEC_U];
#pragma unroll
      for (int u = 0; u < DEC_U; ++u) {
        const int64_t i = i0 + (int64_t)u * DEC_T;
        if (i < n4) {
          const bool obj = (s_m[i >> 3] >> (i & 7)) & 1;
          r[u] = obj ? recon4(it.obase, ro, i * 4) : recon4(it.bbase, rb, i * 4);
        }
      }
#pragma unroll
      for (int u = 0; u < DEC_U; ++u) {
        const int64_t i = i0 + (int64_t)u * DEC_T;
        if (i < n4) __stcs(o4 + i, r[u]);
      }
    }
  } else {
    for (int64_t x = threadIdx.x; x < E; x += DEC_T) {
      const int64_t p = x / C;
      const bool obj = (s_m[p >> 3] >> (p & 7)) & 1;
      out[x] = obj ? recon(it.obase, ro, x) : recon(it.bbase, rb, x);
    }
  }
}

// Plain stitch of latents already in memory (stitcher.cpp:25-37).
__global__ void k_stitch(const float* __restrict__ obj, const uint8_t* __restrict__ om, const float* __restrict__ bg,
                         const uint8_t* __restrict__ sm, int64_t n, int F, int64_t E, int C, int64_t mb,
                         float* __restrict__ out) {
  const int64_t total = n * F * E;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t frame = x / E, e = x - frame * E, p = e / C;
    const bool o = mask_bit(om + frame * mb, p) | mask_bit(sm + frame * mb, p);
    out[x] = o ? obj[x] : bg[x];
  }
}

__global__ void k_solve_alpha(const float* __restrict__ ds, const float* __restrict__ db, int64_t n, int64_t len,
                              float* __restrict__ out, int* __restrict__ bad) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const float* s = ds + r * len;
  const float* b = db + r * len;
  double num = 0.0, den = 0.0;
  for (int64_t i = 0; i < len; ++i) {
    num = fma((double)s[i], (double)b[i], num);
    den = fma((double)b[i], (double)b[i], den);
  }
  if (den == 0.0) {
    atomicExch(bad, 1);
    out[r] = 0.f;
    return;
  }
  out[r] = (float)(num / den);
}

// ---------------------------------------------------------------------------
// host: compress orchestration
// ---------------------------------------------------------------------------
namespace {

struct Geo {
  int F, H, W, C;
  int64_t E, mb;
};

int check_flag(lc_ctx* ctx, DevBuf& flag) {
  int h = 0;
  FC_CUDA(cudaMemcpyAsync(&h, flag.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  return h;
}

void gram(lc_ctx* ctx, const float* lat, int n_items, const Geo& g, double* G) {
  const int FP = (g.F + 7) & ~7;
  const size_t smem = (size_t)(4096 / FP) * (FP + 2) * sizeof(double);
  FC_CUDA(cudaFuncSetAttribute(k_gram, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  KTimer kt(ctx, "gram");
  k_gram<<<n_items, 64, smem, ctx->stream>>>(lat, g.F, g.E, G);
  kt.stop();
  FC_LAUNCH_CHECK();
  count_launch(ctx);
}

// Builds entries for n prompts given maps (host, [n][S][F] in input step
// order) and the device Gram diagonals. Writes out[i], sizes[i].
void assemble(lc_ctx* ctx, const float* lat, const uint8_t* om, const uint8_t* bm, const std::vector<int32_t>& steps_in,
              const Geo& g, const std::vector<int32_t>& maps_h, const double* G_dev, const uint64_t* prompts, int64_t n,
              lc_entry** out, uint64_t* sizes) {
  const int S = (int)steps_in.size();
  const int F = g.F;
  const int64_t E = g.E;
  // sorted step order (codec.cpp:197-199)
  std::vector<int> perm(S);
  std::iota(perm.begin(), perm.end(), 0);
  std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return steps_in[a] < steps_in[b]; });
  // per-entry keys and common key set (codec.cpp:213-220)
  std::vector<std::vector<int>> common(n);
  std::vector<InterItem> items;
  std::vector<int> item_begin(n + 1, 0);
  for (int64_t e = 0; e < n; ++e) {
    item_begin[e] = (int)items.size();
    for (int j = 0; j < F; ++j) {
      bool all = true;
      for (int s = 0; s < S; ++s)
        if (maps_h[((size_t)e * S + s) * F + j] != j) {
          all = false;
          break;
        }
      if (all) {
        common[e].push_back(j);
        if (j > 0) items.push_back(InterItem{(int32_t)e, (int32_t)j});
      }
    }
  }
  item_begin[n] = (int)items.size();
  // Gram diagonals (norms^2 of every frame) to the host
  std::vector<double> diag((size_t)n * S * F);
  {
    DevBuf d((size_t)n * S * F * sizeof(double), ctx->stream);
    k_diag<<<grid_for((int64_t)n * S * F, 256), 256, 0, ctx->stream>>>(G_dev, (int64_t)n * S, F, d.as<double>());
    FC_LAUNCH_CHECK();
    count_launch(ctx);
    FC_CUDA(cudaMemcpyAsync(diag.data(), d.p, diag.size() * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
  }
  // K7 over all (entry, common key) items
  std::vector<InterRes> res(items.size());
  if (!items.empty()) {
    DevBuf di(items.size() * sizeof(InterItem), ctx->stream), dr(items.size() * sizeof(InterRes), ctx->stream),
        dp(S * sizeof(int), ctx->stream);
    FC_CUDA(cudaMemcpyAsync(di.p, items.data(), di.bytes, cudaMemcpyHostToDevice, ctx->stream));
    FC_CUDA(cudaMemcpyAsync(dp.p, perm.data(), dp.bytes, cudaMemcpyHostToDevice, ctx->stream));
    KTimer kt(ctx, "inter");
    k_inter<<<(unsigned)items.size(), INTER_T, 0, ctx->stream>>>(lat, di.as<InterItem>(), S, dp.as<int>(), F, E, G_dev,
                                                                  dr.as<InterRes>());
    FC_LAUNCH_CHECK();
    count_launch(ctx);
    FC_CUDA(cudaMemcpyAsync(res.data(), dr.p, dr.bytes, cudaMemcpyDeviceToHost, ctx->stream));
    sync(ctx);
  }
  auto identical_sim = [](double ss) { return ss == 0.0 ? 1.0 : ss / (std::sqrt(ss) * std::sqrt(ss)); };
  // ---- per entry: base selection + assembly metadata ----
  std::vector<std::shared_ptr<EntryData>> ents(n);
  std::vector<FrameJob> fjobs;
  std::vector<ByteJob> bjobs;
  std::vector<Recipe> all_recipes;
  std::vector<std::pair<size_t, size_t>> recipe_span(n);
  for (int64_t e = 0; e < n; ++e) {
    const auto& cm = common[e];
    const int i0 = item_begin[e];
    auto in_common = [&](int m) { return std::binary_search(cm.begin(), cm.end(), m); };
    auto item_of = [&](int m) -> const InterRes* {
      // items for this entry are in ascending m (skipping 0)
      int lo = i0, hi = item_begin[e + 1];
      while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (items[mid].m < m) lo = mid + 1; else hi = mid;
      }
      return (lo < item_begin[e + 1] && items[lo].m == m) ? &res[lo] : nullptr;
    };
    auto mapv = [&](int si, int j) { return maps_h[((size_t)e * S + perm[si]) * F + j]; };
    auto dg = [&](int si, int m) { return diag[((size_t)e * S + perm[si]) * F + m]; };
    // choose base (codec.cpp:240-259); a single step is its own base
    int best_b = 0;
    if (S > 1) {
      double best_score = -2.0;
      for (int b = 0; b < S; ++b) {
        // a non-finite trial reconstruction makes decompress_step throw
        for (int c = i0; c < item_begin[e + 1]; ++c)
          for (int s = 0; s < S; ++s)
            if (s != b && res[c].nz[b] && std::isfinite(res[c].alpha[s][b]) && res[c].nonfinite[s][b])
              raise(LC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
        double sum = 0.0;
        uint64_t count = 0;
        for (int si = 0; si < S; ++si) {
          for (int j = 0; j < F; ++j) {
            const int m = mapv(si, j);
            double sim;
            const InterRes* r = (m > 0 && in_common(m)) ? item_of(m) : nullptr;
            if (r && r->nz[b] && si != b && std::isfinite(r->alpha[si][b])) sim = r->sim[si][b];
            else sim = identical_sim(dg(si, m));
            sum += sim;
            ++count;
          }
        }
        const double score = sum / (double)count;
        if (score > best_score) {
          best_score = score;
          best_b = b;
        }
      }
    }
    auto d = std::make_shared<EntryData>();
    d->ctx = ctx;
    d->prompt = prompts[e];
    d->base_step = steps_in[perm[best_b]];
    d->F = F; d->H = g.H; d->W = g.W; d->C = g.C; d->E = E; d->mb = g.mb;
    for (int m : cm) {
      if (m == 0) continue;
      if (item_of(m)->nz[best_b]) d->diff_idx.push_back(m);
    }
    const int nd = (int)d->diff_idx.size();
    d->steps.resize(S);
    d->maps.resize(S);
    d->extra_idx.resize(S);
    d->alphas.resize(S);
    for (int si = 0; si < S; ++si) {
      d->steps[si] = steps_in[perm[si]];
      d->maps[si].resize(F);
      for (int j = 0; j < F; ++j) d->maps[si][j] = mapv(si, j);
      for (int m = 1; m < F; ++m) {
        if (d->maps[si][m] != m) continue;
        if (!in_common(m)) {
          d->extra_idx[si].push_back(m);
          continue;
        }
        const InterRes* r = item_of(m);
        if (!r->nz[best_b]) {
          if (r->nz[si]) d->extra_idx[si].push_back(m);
          continue;
        }
        if (si == best_b) {
          if (!r->exact[si]) d->extra_idx[si].push_back(m);
        } else if (!std::isfinite(r->alpha[si][best_b])) {
          d->extra_idx[si].push_back(m);
        }
      }
      if (si != best_b) {
        d->alphas[si].resize(nd);
        for (int t = 0; t < nd; ++t) {
          const float a = item_of(d->diff_idx[t])->alpha[si][best_b];
          d->alphas[si][t] = std::isfinite(a) ? a : 0.0f;
        }
      }
    }
    // device layout
    int64_t off = 0;
    d->first_off.resize(S);
    for (int si = 0; si < S; ++si) { d->first_off[si] = off; off += E; }
    d->diff_off.resize(nd);
    for (int t = 0; t < nd; ++t) { d->diff_off[t] = off; off += E; }
    d->extra_off.resize(S);
    for (int si = 0; si < S; ++si)
      for (size_t x = 0; x < d->extra_idx[si].size(); ++x) { d->extra_off[si].push_back(off); off += E; }
    int64_t bytes = ((off * 4 + 15) / 16) * 16;
    d->mask_off = bytes;
    bytes += ((2 * F * g.mb + 15) / 16) * 16;
    d->recipe_off = bytes;
    bytes += (int64_t)S * F * sizeof(Recipe);
    d->dev_bytes = (size_t)bytes;
    FC_CUDA(cudaMallocAsync((void**)&d->dev, d->dev_bytes, ctx->stream));
    float* fb = reinterpret_cast<float*>(d->dev);
    const float* latE = lat + (int64_t)e * S * F * E;
    auto frame_ptr = [&](int si, int m) { return latE + ((int64_t)perm[si] * F + m) * E; };
    for (int si = 0; si < S; ++si) fjobs.push_back(FrameJob{fb + d->first_off[si], frame_ptr(si, 0), nullptr});
    const int bsi = best_b;
    for (int t = 0; t < nd; ++t)
      fjobs.push_back(FrameJob{fb + d->diff_off[t], frame_ptr(bsi, d->diff_idx[t]), frame_ptr(bsi, 0)});
    for (int si = 0; si < S; ++si)
      for (size_t x = 0; x < d->extra_idx[si].size(); ++x)
        fjobs.push_back(FrameJob{fb + d->extra_off[si][x], frame_ptr(si, d->extra_idx[si][x]), nullptr});
    bjobs.push_back(ByteJob{d->dev + d->mask_off, om + (int64_t)e * F * g.mb, (int64_t)F * g.mb});
    bjobs.push_back(ByteJob{d->dev + d->mask_off + F * g.mb, bm + (int64_t)e * F * g.mb, (int64_t)F * g.mb});
    // recipes: decompress_step (codec.cpp:271-299) resolved per frame
    recipe_span[e].first = all_recipes.size();
    for (int si = 0; si < S; ++si) {
      std::vector<Recipe> key_rec(F);
      for (int m = 0; m < F; ++m) {
        if (d->maps[si][m] != m) continue;
        Recipe r{0, 0.f, d->first_off[si], 0};
        if (m != 0) {
          auto xi = std::lower_bound(d->extra_idx[si].begin(), d->extra_idx[si].end(), m);
          if (xi != d->extra_idx[si].end() && *xi == m) {
            r.a = d->extra_off[si][xi - d->extra_idx[si].begin()];
          } else {
            auto di = std::lower_bound(d->diff_idx.begin(), d->diff_idx.end(), m);
            if (di != d->diff_idx.end() && *di == m) {
              const size_t t = di - d->diff_idx.begin();
              r.b = d->diff_off[t];
              if (si == best_b) r.kind = 1;
              else {
                r.kind = 2;
                r.alpha = d->alphas[si][t];
              }
            }
          }
        }
        key_rec[m] = r;
      }
      for (int j = 0; j < F; ++j) all_recipes.push_back(key_rec[d->maps[si][j]]);
    }
    recipe_span[e].second = all_recipes.size();
    ents[e] = d;
  }
  // ---- K8: pack frames, masks, recipes ----
  DevBuf rstage(all_recipes.size() * sizeof(Recipe), ctx->stream);
  if (!all_recipes.empty())
    FC_CUDA(cudaMemcpyAsync(rstage.p, all_recipes.data(), rstage.bytes, cudaMemcpyHostToDevice, ctx->stream));
  for (int64_t e = 0; e < n; ++e)
    bjobs.push_back(ByteJob{ents[e]->dev + ents[e]->recipe_off, rstage.as<uint8_t>() + recipe_span[e].first * sizeof(Recipe),
                            (int64_t)((recipe_span[e].second - recipe_span[e].first) * sizeof(Recipe))});
  DevBuf dfj(fjobs.size() * sizeof(FrameJob), ctx->stream), dbj(bjobs.size() * sizeof(ByteJob), ctx->stream);
  FC_CUDA(cudaMemcpyAsync(dfj.p, fjobs.data(), dfj.bytes, cudaMemcpyHostToDevice, ctx->stream));
  FC_CUDA(cudaMemcpyAsync(dbj.p, bjobs.data(), dbj.bytes, cudaMemcpyHostToDevice, ctx->stream));
  KTimer ktp(ctx, "pack");
  for (size_t j0 = 0; j0 < fjobs.size(); j0 += 65535) {
    const unsigned cnt = (unsigned)std::min<size_t>(65535, fjobs.size() - j0);
    k_pack_frames<<<dim3(grid_for(E, 256, 64), cnt), 256, 0, ctx->stream>>>(dfj.as<FrameJob>() + j0, E);
    FC_LAUNCH_CHECK();
  }
  for (size_t j0 = 0; j0 < bjobs.size(); j0 += 65535) {
    const unsigned cnt = (unsigned)std::min<size_t>(65535, bjobs.size() - j0);
    k_pack_bytes<<<dim3(8, cnt), 256, 0, ctx->stream>>>(dbj.as<ByteJob>() + j0);
    FC_LAUNCH_CHECK();
  }
  ktp.stop();
  count_launch(ctx, 2);
  sync(ctx);
  for (int64_t e = 0; e < n; ++e) {
    std::vector<int> sel(S);
    std::iota(sel.begin(), sel.end(), 0);
    out[e] = make_entry_view(ents[e], std::move(sel));
    if (sizes) sizes[e] = entry_compressed_size(out[e]);
  }
}

void validate_geometry(int S, int F, int H, int W, int C, const int32_t* steps) {
  if (H <= 0 || W <= 0 || C <= 0) raise(LC_ERR_INVALID_ARGUMENT, "Frame: dimensions must be positive");
  if (F <= 0) raise(LC_ERR_INVALID_ARGUMENT, "LatentState: needs at least one frame");
  if (S <= 0) raise(LC_ERR_INVALID_ARGUMENT, "inter_compress: empty step list");
  FC_REQUIRE(S <= MAXS, "at most 8 steps per entry");
  FC_REQUIRE(F <= 256, "at most 256 frames per latent");
  for (int s = 0; s < S; ++s)
    if (steps[s] < 1 || steps[s] > 50) raise(LC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
}

void check_distinct_steps(int S, const int32_t* steps) {
  std::vector<int> v(steps, steps + S);
  std::sort(v.begin(), v.end());
  for (int i = 1; i < S; ++i)
    if (v[i] == v[i - 1]) raise(LC_ERR_INVALID_ARGUMENT, "inter_compress: duplicate step");
}

}  // namespace

void launch_decompress(lc_ctx* ctx, const std::vector<const EntryData*>& ents, const std::vector<int>& sidx, float* out,
                       const int32_t*) {
  if (ents.empty()) return;
  const EntryData* d0 = ents[0];
  const int F = d0->F;
  const int64_t E = d0->E;
  std::vector<DecItem> items(ents.size());
  for (size_t i = 0; i < ents.size(); ++i)
    items[i] = DecItem{ents[i]->fbase(), ents[i]->recipes(sidx[i]), out + (int64_t)i * F * E};
  DevBuf di(items.size() * sizeof(DecItem), ctx->stream);
  FC_CUDA(cudaMemcpyAsync(di.p, items.data(), di.bytes, cudaMemcpyHostToDevice, ctx->stream));
  KTimer kt(ctx, "decompress");
  k_decompress<<<(unsigned)(items.size() * F), DEC_T, 0, ctx->stream>>>(di.as<DecItem>(), F, E);
  kt.stop();
  FC_LAUNCH_CHECK();
  count_launch(ctx);
}

}  // namespace fc

using namespace fc;

// ---------------------------------------------------------------------------
// wire format (serialize_entry / deserialize_entry, codec.cpp:358-473)
// ---------------------------------------------------------------------------
namespace {

struct Writer {
  uint8_t* p;
  uint64_t cap, n = 0;
  void put(const void* s, uint64_t k) {
    if (p && n + k <= cap) memcpy(p + n, s, k);
    n += k;
  }
  void u8(uint8_t v) { put(&v, 1); }
  void u16(uint16_t v) {
    uint8_t t[2] = {(uint8_t)v, (uint8_t)(v >> 8)};
    put(t, 2);
  }
  void u64(uint64_t v) {
    uint8_t t[8];
    for (int i = 0; i < 8; ++i) t[i] = (uint8_t)(v >> (8 * i));
    put(t, 8);
  }
  void f32s(const float* v, int64_t k) { put(v, 4ull * k); }  // little-endian host
};

struct Reader {
  const uint8_t* p;
  uint64_t n, pos = 0;
  void need(uint64_t k) {
    if (pos + k > n) raise(LC_ERR_SNAPSHOT, "truncated input at byte " + std::to_string(pos));
  }
  uint8_t u8() { need(1); return p[pos++]; }
  uint16_t u16() { need(2); uint16_t v = (uint16_t)(p[pos] | (p[pos + 1] << 8)); pos += 2; return v; }
  uint64_t u64() {
    need(8);
    uint64_t v = 0;
    for (int i = 0; i < 8; ++i) v |= (uint64_t)p[pos + i] << (8 * i);
    pos += 8;
    return v;
  }
  const uint8_t* bytes(uint64_t k) { need(k); const uint8_t* r = p + pos; pos += k; return r; }
};

bool all_finite(const float* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

}  // namespace

extern "C" {

lc_status lc_select_keyframes(lc_ctx* ctx, const float* latents, int64_t n, int F, int H, int W, int C, double thr,
                              int32_t* map) {
  LC_API_BEGIN
  if (H <= 0 || W <= 0 || C <= 0) raise(LC_ERR_INVALID_ARGUMENT, "Frame: dimensions must be positive");
  if (F <= 0) raise(LC_ERR_INVALID_ARGUMENT, "LatentState: needs at least one frame");
  FC_REQUIRE(F <= 256, "at most 256 frames");
  if (thr <= 0.0 || thr > 1.0) raise(LC_ERR_INVALID_ARGUMENT, "select_keyframes: threshold must be in (0, 1]");
  if (n <= 0) return LC_OK;
  DeviceGuard dg(ctx->device);
  const int64_t E = (int64_t)H * W * C;
  InArg<float> lat(ctx, latents, (size_t)n * F * E);
  OutArg<int32_t> om(ctx, map, (size_t)n * F);
  DevBuf bad(sizeof(int), ctx->stream);
  FC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
  k_nonfinite<<<grid_for(n * F * E, 256, 4096), 256, 0, ctx->stream>>>(lat.dev, n * F * E, bad.as<int>());
  FC_LAUNCH_CHECK();
  DevBuf G((size_t)n * F * F * sizeof(double), ctx->stream);
  Geo g{F, H, W, C, E, ((int64_t)H * W + 7) / 8};
  gram(ctx, lat.dev, (int)n, g, G.as<double>());
  if (check_flag(ctx, bad)) raise(LC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
  k_select<<<grid_for(n, 64), 64, 0, ctx->stream>>>(G.as<double>(), (int)n, F, thr, om.dev, bad.as<int>());
  FC_LAUNCH_CHECK();
  count_launch(ctx, 2);
  om.finish(ctx);
  if (check_flag(ctx, bad)) raise(LC_ERR_INVALID_ARGUMENT, "cosine_similarity: zero-norm operand");
  LC_API_END
}

lc_status lc_solve_alpha_batch(lc_ctx* ctx, const float* ds, const float* db, int64_t n, int64_t len, float* out) {
  LC_API_BEGIN
  if (n <= 0) return LC_OK;
  DeviceGuard dg(ctx->device);
  InArg<float> a(ctx, ds, (size_t)n * len), b(ctx, db, (size_t)n * len);
  OutArg<float> o(ctx, out, (size_t)n);
  DevBuf bad(sizeof(int), ctx->stream);
  FC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
  k_solve_alpha<<<grid_for(n, 128), 128, 0, ctx->stream>>>(a.dev, b.dev, n, len, o.dev, bad.as<int>());
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  o.finish(ctx);
  if (check_flag(ctx, bad)) raise(LC_ERR_DEGENERATE_BASE, "solve_alpha: base differential is identically zero");
  LC_API_END
}

lc_status lc_compress_batch(lc_ctx* ctx, const float* latents, const int32_t* steps, int S, int F, int H, int W, int C,
                            const uint8_t* obj_masks, const uint8_t* bg_masks, double thr, const uint64_t* prompts,
                            int64_t n, lc_entry** out, uint64_t* sizes) {
  LC_API_BEGIN
  FC_REQUIRE(steps && out && prompts, "lc_compress_batch: null argument");
  validate_geometry(S, F, H, W, C, steps);
  if (thr <= 0.0 || thr > 1.0) raise(LC_ERR_INVALID_ARGUMENT, "select_keyframes: threshold must be in (0, 1]");
  if (n <= 0) return LC_OK;
  DeviceGuard dg(ctx->device);
  const int64_t E = (int64_t)H * W * C;
  Geo g{F, H, W, C, E, ((int64_t)H * W + 7) / 8};
  InArg<float> lat(ctx, latents, (size_t)n * S * F * E);
  InArg<uint8_t> om(ctx, obj_masks, (size_t)n * F * g.mb), bm(ctx, bg_masks, (size_t)n * F * g.mb);
  DevBuf bad(sizeof(int), ctx->stream);
  FC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
  k_nonfinite<<<grid_for(n * S * F * E, 256, 8192), 256, 0, ctx->stream>>>(lat.dev, n * S * F * E, bad.as<int>());
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  // K5 + K6: key frames of every (prompt, step)
  DevBuf G((size_t)n * S * F * F * sizeof(double), ctx->stream);
  gram(ctx, lat.dev, (int)(n * S), g, G.as<double>());
  if (check_flag(ctx, bad)) raise(LC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
  DevBuf maps((size_t)n * S * F * sizeof(int32_t), ctx->stream);
  k_select<<<grid_for(n * S, 64), 64, 0, ctx->stream>>>(G.as<double>(), (int)(n * S), F, thr, maps.as<int32_t>(),
                                                        bad.as<int>());
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  std::vector<int32_t> maps_h((size_t)n * S * F);
  FC_CUDA(cudaMemcpyAsync(maps_h.data(), maps.p, maps.bytes, cudaMemcpyDeviceToHost, ctx->stream));
  if (check_flag(ctx, bad)) raise(LC_ERR_INVALID_ARGUMENT, "cosine_similarity: zero-norm operand");
  check_distinct_steps(S, steps);
  std::vector<int32_t> st(steps, steps + S);
  assemble(ctx, lat.dev, om.dev, bm.dev, st, g, maps_h, G.as<double>(), prompts, n, out, sizes);
  LC_API_END
}

lc_status lc_inter_compress(lc_ctx* ctx, const float* latents, const int32_t* maps, const int32_t* steps, int S, int F,
                            int H, int W, int C, const uint8_t* obj_masks, const uint8_t* bg_masks, uint64_t prompt,
                            lc_entry** out) {
  LC_API_BEGIN
  FC_REQUIRE(steps && out && maps, "lc_inter_compress: null argument");
  validate_geometry(S, F, H, W, C, steps);
  check_distinct_steps(S, steps);
  DeviceGuard dg(ctx->device);
  const int64_t E = (int64_t)H * W * C;
  Geo g{F, H, W, C, E, ((int64_t)H * W + 7) / 8};
  std::vector<int32_t> maps_h((size_t)S * F);
  if (is_device_ptr(maps)) FC_CUDA(cudaMemcpy(maps_h.data(), maps, maps_h.size() * 4, cudaMemcpyDeviceToHost));
  else memcpy(maps_h.data(), maps, maps_h.size() * 4);
  for (int s = 0; s < S; ++s)
    for (int j = 0; j < F; ++j) {
      const int m = maps_h[(size_t)s * F + j];
      FC_REQUIRE(m >= 0 && m <= j && maps_h[(size_t)s * F + m] == m && maps_h[(size_t)s * F] == 0,
                 "KeyFrameMap: invalid mapping");
    }
  InArg<float> lat(ctx, latents, (size_t)S * F * E);
  InArg<uint8_t> om(ctx, obj_masks, (size_t)F * g.mb), bm(ctx, bg_masks, (size_t)F * g.mb);
  DevBuf G((size_t)S * F * F * sizeof(double), ctx->stream);
  gram(ctx, lat.dev, S, g, G.as<double>());
  std::vector<int32_t> st(steps, steps + S);
  assemble(ctx, lat.dev, om.dev, bm.dev, st, g, maps_h, G.as<double>(), &prompt, 1, out, nullptr);
  LC_API_END
}

lc_status lc_entry_release(lc_entry* e) {
  LC_API_BEGIN
  delete e;
  LC_API_END
}

lc_status lc_entry_get_info(lc_entry* e, lc_entry_info* o) {
  LC_API_BEGIN
  FC_REQUIRE(e && o, "null argument");
  const EntryData& d = *e->d;
  memset(o, 0, sizeof *o);
  o->prompt = d.prompt;
  o->base_step = d.base_step;
  o->n_steps = (int)e->sel.size();
  o->F = d.F; o->H = d.H; o->W = d.W; o->C = d.C;
  o->n_diff = d.n_diff();
  o->shared_bytes = d.shared_bytes();
  for (size_t i = 0; i < e->sel.size() && i < 8; ++i) {
    o->steps[i] = d.steps[e->sel[i]];
    o->n_extra[i] = (int)d.extra_idx[e->sel[i]].size();
    o->private_bytes[i] = d.private_bytes(e->sel[i]);
  }
  o->compressed_size = entry_compressed_size(e);
  LC_API_END
}

lc_status lc_entry_export(lc_entry* e, uint8_t* bytes, uint64_t cap, uint64_t* len) {
  LC_API_BEGIN
  FC_REQUIRE(e && len, "null argument");
  const EntryData& d = *e->d;
  const uint64_t total = entry_compressed_size(e);
  *len = total;
  if (!bytes) return LC_OK;
  FC_REQUIRE(cap >= total, "lc_entry_export: buffer too small");
  DeviceGuard dg(d.ctx->device);
  std::vector<uint8_t> img(d.dev_bytes);
  FC_CUDA(cudaMemcpyAsync(img.data(), d.dev, d.dev_bytes, cudaMemcpyDeviceToHost, d.ctx->stream));
  sync(d.ctx);
  const float* fb = reinterpret_cast<const float*>(img.data());
  Writer w{bytes, cap};
  w.u64(d.prompt);
  w.u8((uint8_t)d.base_step);
  w.u8((uint8_t)e->sel.size());
  w.u16((uint16_t)d.n_diff());
  w.u16((uint16_t)d.F);
  w.u16((uint16_t)d.H);
  w.u16((uint16_t)d.W);
  w.u16((uint16_t)d.C);
  for (int si : e->sel) {
    w.u8((uint8_t)d.steps[si]);
    w.f32s(fb + d.first_off[si], d.E);
    for (int j = 0; j < d.F; ++j) w.u16((uint16_t)d.maps[si][j]);
    if (d.steps[si] != d.base_step) w.f32s(d.alphas[si].data(), (int64_t)d.alphas[si].size());
    w.u16((uint16_t)d.extra_idx[si].size());
    for (size_t x = 0; x < d.extra_idx[si].size(); ++x) {
      w.u16((uint16_t)d.extra_idx[si][x]);
      w.f32s(fb + d.extra_off[si][x], d.E);
    }
  }
  for (int t = 0; t < d.n_diff(); ++t) {
    w.u16((uint16_t)d.diff_idx[t]);
    w.f32s(fb + d.diff_off[t], d.E);
  }
  w.put(img.data() + d.mask_off, 2ull * d.F * d.mb);
  if (w.n != total) raise(LC_ERR_INTERNAL, "lc_entry_export: size accounting mismatch");
  LC_API_END
}

lc_status lc_entry_import(lc_ctx* ctx, const uint8_t* bytes, uint64_t len, lc_entry** out) {
  LC_API_BEGIN
  FC_REQUIRE(ctx && bytes && out, "null argument");
  DeviceGuard dg(ctx->device);
  Reader r{bytes, len};
  auto d = std::make_shared<EntryData>();
  d->ctx = ctx;
  d->prompt = r.u64();
  const int base = r.u8();
  const int ns = r.u8();
  const int nd = r.u16();
  d->F = r.u16();
  d->H = r.u16();
  d->W = r.u16();
  d->C = r.u16();
  if (ns < 1 || d->F < 1 || d->H < 1 || d->W < 1 || d->C < 1) raise(LC_ERR_SNAPSHOT, "invalid entry header at byte 0");
  if (base < 1 || base > 50) raise(LC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
  d->base_step = base;
  d->E = (int64_t)d->H * d->W * d->C;
  d->mb = ((int64_t)d->H * d->W + 7) / 8;
  const int64_t E = d->E;
  std::vector<const uint8_t*> firsts(ns), raw_alpha(ns, nullptr);
  std::vector<std::vector<const uint8_t*>> extras(ns);
  d->steps.resize(ns);
  d->maps.resize(ns);
  d->extra_idx.resize(ns);
  d->alphas.resize(ns);
  for (int s = 0; s < ns; ++s) {
    const uint64_t step_pos = r.pos;
    const int step = r.u8();
    if (step < 1 || step > 50) raise(LC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
    d->steps[s] = step;
    firsts[s] = r.bytes(4ull * E);
    d->maps[s].resize(d->F);
    for (int j = 0; j < d->F; ++j) {
      d->maps[s][j] = r.u16();
      if (d->maps[s][j] >= d->F) raise(LC_ERR_SNAPSHOT, "key frame map index out of range at byte " + std::to_string(step_pos));
    }
    if (step != base) raw_alpha[s] = r.bytes(4ull * nd);
    const int nx = r.u16();
    std::vector<std::pair<int, const uint8_t*>> xs;
    for (int x = 0; x < nx; ++x) {
      const int m = r.u16();
      if (m >= d->F) raise(LC_ERR_SNAPSHOT, "extra frame index out of range at byte " + std::to_string(step_pos));
      const uint8_t* fr = r.bytes(4ull * E);
      bool dup = false;
      for (auto& pr : xs) dup |= pr.first == m;
      if (!dup) xs.emplace_back(m, fr);  // std::map::emplace keeps the first
    }
    std::sort(xs.begin(), xs.end(), [](auto& a, auto& b) { return a.first < b.first; });
    for (auto& pr : xs) {
      d->extra_idx[s].push_back(pr.first);
      extras[s].push_back(pr.second);
    }
    if (s > 0 && !(d->steps[s - 1] < step)) raise(LC_ERR_SNAPSHOT, "steps out of order at byte " + std::to_string(step_pos));
  }
  std::vector<const uint8_t*> diffs(nd);
  for (int t = 0; t < nd; ++t) {
    const uint64_t pos = r.pos;
    const int m = r.u16();
    if (m < 1 || m >= d->F) raise(LC_ERR_SNAPSHOT, "diff index out of range at byte " + std::to_string(pos));
    d->diff_idx.push_back(m);
    diffs[t] = r.bytes(4ull * E);
  }
  for (int t = 1; t < nd; ++t) {
    if (d->diff_idx[t] < d->diff_idx[t - 1]) raise(LC_ERR_SNAPSHOT, "diff indices out of order at byte " + std::to_string(r.pos));
    if (d->diff_idx[t] == d->diff_idx[t - 1]) raise(LC_ERR_SNAPSHOT, "duplicate diff index");
  }
  for (int s = 0; s < ns; ++s) {
    if (d->steps[s] == base) continue;
    d->alphas[s].resize(nd);
    if (nd) memcpy(d->alphas[s].data(), raw_alpha[s], 4ull * nd);
  }
  const uint8_t* masks = r.bytes(2ull * d->F * d->mb);
  if (r.pos != len) raise(LC_ERR_SNAPSHOT, "trailing bytes at byte " + std::to_string(r.pos));
  // host image -> device
  int64_t off = 0;
  d->first_off.resize(ns);
  for (int s = 0; s < ns; ++s) { d->first_off[s] = off; off += E; }
  d->diff_off.resize(nd);
  for (int t = 0; t < nd; ++t) { d->diff_off[t] = off; off += E; }
  d->extra_off.resize(ns);
  for (int s = 0; s < ns; ++s)
    for (size_t x = 0; x < d->extra_idx[s].size(); ++x) { d->extra_off[s].push_back(off); off += E; }
  int64_t bytes_n = ((off * 4 + 15) / 16) * 16;
  d->mask_off = bytes_n;
  bytes_n += ((2 * d->F * d->mb + 15) / 16) * 16;
  d->recipe_off = bytes_n;
  bytes_n += (int64_t)ns * d->F * sizeof(Recipe);
  d->dev_bytes = (size_t)bytes_n;
  std::vector<uint8_t> img(d->dev_bytes, 0);
  for (int s = 0; s < ns; ++s) memcpy(img.data() + 4 * d->first_off[s], firsts[s], 4ull * E);
  for (int t = 0; t < nd; ++t) memcpy(img.data() + 4 * d->diff_off[t], diffs[t], 4ull * E);
  for (int s = 0; s < ns; ++s)
    for (size_t x = 0; x < extras[s].size(); ++x) memcpy(img.data() + 4 * d->extra_off[s][x], extras[s][x], 4ull * E);
  if (!all_finite(reinterpret_cast<const float*>(img.data()), off)) {
    // diffs are not Frames (no finite check) in the reference; only firsts/extras are
    for (int s = 0; s < ns; ++s) {
      if (!all_finite(reinterpret_cast<const float*>(img.data() + 4 * d->first_off[s]), E))
        raise(LC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
      for (size_t x = 0; x < extras[s].size(); ++x)
        if (!all_finite(reinterpret_cast<const float*>(img.data() + 4 * d->extra_off[s][x]), E))
          raise(LC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
    }
  }
  memcpy(img.data() + d->mask_off, masks, 2ull * d->F * d->mb);
  Recipe* rec = reinterpret_cast<Recipe*>(img.data() + d->recipe_off);
  for (int s = 0; s < ns; ++s) {
    std::vector<Recipe> key_rec(d->F);
    for (int m = 0; m < d->F; ++m) {
      Recipe rr{0, 0.f, d->first_off[s], 0};
      if (m != 0) {
        auto xi = std::lower_bound(d->extra_idx[s].begin(), d->extra_idx[s].end(), m);
        if (xi != d->extra_idx[s].end() && *xi == m) {
          rr.a = d->extra_off[s][xi - d->extra_idx[s].begin()];
        } else {
          auto di = std::lower_bound(d->diff_idx.begin(), d->diff_idx.end(), m);
          if (di != d->diff_idx.end() && *di == m) {
            const size_t t = di - d->diff_idx.begin();
            rr.b = d->diff_off[t];
            if (d->steps[s] == base) rr.kind = 1;
            else {
              rr.kind = 2;
              rr.alpha = d->alphas[s][t];
            }
          }
        }
      }
      key_rec[m] = rr;
    }
    // a non-key frame maps to a key; decompress copies that key's reconstruction
    for (int j = 0; j < d->F; ++j) rec[(size_t)s * d->F + j] = key_rec[d->maps[s][j]];
  }
  FC_CUDA(cudaMallocAsync((void**)&d->dev, d->dev_bytes, ctx->stream));
  FC_CUDA(cudaMemcpyAsync(d->dev, img.data(), d->dev_bytes, cudaMemcpyHostToDevice, ctx->stream));
  sync(ctx);
  std::vector<int> sel(ns);
  std::iota(sel.begin(), sel.end(), 0);
  *out = make_entry_view(d, std::move(sel));
  LC_API_END
}

lc_status lc_decompress_batch(lc_ctx* ctx, lc_entry* const* entries, const int32_t* steps, int64_t n, float* out_dev) {
  LC_API_BEGIN
  if (n <= 0) return LC_OK;
  FC_REQUIRE(entries && steps && out_dev, "null argument");
  FC_REQUIRE(is_device_ptr(out_dev), "lc_decompress_batch: out_dev must be device memory");
  DeviceGuard dg(ctx->device);
  std::vector<const EntryData*> ents(n);
  std::vector<int> sidx(n);
  for (int64_t i = 0; i < n; ++i) {
    const lc_entry* e = entries[i];
    FC_REQUIRE(e, "null entry");
    if (steps[i] < 1 || steps[i] > 50) raise(LC_ERR_INVALID_ARGUMENT, "StepId: value out of range 1..50");
    int si = -1;
    for (int k : e->sel)
      if (e->d->steps[k] == steps[i]) si = k;
    if (si < 0) raise(LC_ERR_STEP_NOT_CACHED, "step " + std::to_string(steps[i]) + " not in entry");
    if (i > 0) FC_REQUIRE(e->d->F == ents[0]->F && e->d->E == ents[0]->E, "lc_decompress_batch: mixed shapes");
    ents[i] = e->d.get();
    sidx[i] = si;
  }
  launch_decompress(ctx, ents, sidx, out_dev);
  sync(ctx);
  LC_API_END
}

lc_status lc_decompress_stitch_batch(lc_ctx* ctx, lc_entry* const* oe, lc_entry* const* be, const int32_t* steps, int64_t n,
                                     float* out_dev) {
  LC_API_BEGIN
  if (n <= 0) return LC_OK;
  FC_REQUIRE(oe && be && steps && out_dev, "null argument");
  FC_REQUIRE(is_device_ptr(out_dev), "lc_decompress_stitch_batch: out_dev must be device memory");
  DeviceGuard dg(ctx->device);
  std::vector<StitchItem> items(n);
  const EntryData* d0 = oe[0]->d.get();
  for (int64_t i = 0; i < n; ++i) {
    const lc_entry* pair[2] = {oe[i], be[i]};
    int si[2] = {-1, -1};
    for (int t = 0; t < 2; ++t) {
      for (int k : pair[t]->sel)
        if (pair[t]->d->steps[k] == steps[i]) si[t] = k;
      if (si[t] < 0) raise(LC_ERR_STEP_NOT_CACHED, "step " + std::to_string(steps[i]) + " not in entry");
    }
    const EntryData* a = pair[0]->d.get();
    const EntryData* b = pair[1]->d.get();
    if (a->F != b->F || a->H != b->H || a->W != b->W || a->C != b->C)
      raise(LC_ERR_INVALID_ARGUMENT, "stitch: latent shape mismatch");
    FC_REQUIRE(a->F == d0->F && a->E == d0->E && a->C == d0->C, "lc_decompress_stitch_batch: mixed shapes");
    items[i] = StitchItem{a->fbase(), a->recipes(si[0]), b->fbase(), b->recipes(si[1]), a->obj_masks(), b->obj_masks(),
                          out_dev + i * (int64_t)a->F * a->E};
  }
  DevBuf di(items.size() * sizeof(StitchItem), ctx->stream);
  FC_CUDA(cudaMemcpyAsync(di.p, items.data(), di.bytes, cudaMemcpyHostToDevice, ctx->stream));
  KTimer kt(ctx, "decompress_stitch");
  k_decompress_stitch<<<(unsigned)(n * d0->F), DEC_T, (size_t)d0->mb, ctx->stream>>>(di.as<StitchItem>(), d0->F, d0->E,
                                                                                     d0->C, d0->mb);
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  sync(ctx);
  LC_API_END
}

lc_status lc_stitch_batch(lc_ctx* ctx, const float* obj, const uint8_t* om, const float* bg, const uint8_t* sm, int64_t n,
                          int F, int H, int W, int C, float* out) {
  LC_API_BEGIN
  if (H <= 0 || W <= 0 || C <= 0) raise(LC_ERR_INVALID_ARGUMENT, "Frame: dimensions must be positive");
  if (F <= 0) raise(LC_ERR_INVALID_ARGUMENT, "LatentState: needs at least one frame");
  if (n <= 0) return LC_OK;
  DeviceGuard dg(ctx->device);
  const int64_t E = (int64_t)H * W * C, mb = ((int64_t)H * W + 7) / 8;
  InArg<float> a(ctx, obj, (size_t)n * F * E), b(ctx, bg, (size_t)n * F * E);
  InArg<uint8_t> m1(ctx, om, (size_t)n * F * mb), m2(ctx, sm, (size_t)n * F * mb);
  OutArg<float> o(ctx, out, (size_t)n * F * E);
  DevBuf bad(sizeof(int), ctx->stream);
  FC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
  k_nonfinite<<<grid_for(n * F * E, 256, 4096), 256, 0, ctx->stream>>>(a.dev, n * F * E, bad.as<int>());
  k_nonfinite<<<grid_for(n * F * E, 256, 4096), 256, 0, ctx->stream>>>(b.dev, n * F * E, bad.as<int>());
  k_stitch<<<grid_for(n * F * E, 256, 1 << 20), 256, 0, ctx->stream>>>(a.dev, m1.dev, b.dev, m2.dev, n, F, E, C, mb, o.dev);
  FC_LAUNCH_CHECK();
  count_launch(ctx, 3);
  o.finish(ctx);
  if (check_flag(ctx, bad)) raise(LC_ERR_INVALID_ARGUMENT, "Frame: non-finite element");
  LC_API_END
}

}  // extern "C"
