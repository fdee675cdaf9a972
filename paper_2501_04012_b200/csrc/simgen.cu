// simgen.cu — on-device synthetic workload generator (
// SPEC.md:564-632, simgen.hpp:25-93). The reference declares simgen but
// ships no code; the SPEC fixes only its properties, so the generator is
// defined here and restated line for line in
// oracle/lc_oracle.c (orc_synth_*), which the GPU output matches bit for bit.
//
// Randomness is counter-based so every element is generated independently:
//   ctr(s, i) = hash_combine(s, i)                          (rng.hpp:25-31)
//   U(s, i)   = (ctr(s, i) >> 11) * 2^-53                   (rng.hpp:71 form)
//   N(s, i)   = ((U(s,4i) + U(s,4i+1)) + (U(s,4i+2) + U(s,4i+3)) - 2) * sqrt(3)
// (Irwin-Hall, unit variance; only correctly rounded adds/muls, so CPU and
// GPU agree bitwise — Box-Muller's log/sin/cos would not.)
#include <cmath>

#include "common.cuh"

namespace fc {
namespace sg {

__host__ __device__ __forceinline__ uint64_t hash_combine(uint64_t a, uint64_t b) {
  uint64_t z = a ^ (b + 0x9e3779b97f4a7c15ull + (a << 6) + (a >> 2));
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double U(uint64_t s, uint64_t i) {
  return __dmul_rn((double)(hash_combine(s, i) >> 11), 0x1.0p-53);
}
__device__ __forceinline__ double N(uint64_t s, uint64_t i) {
  const double a = __dadd_rn(U(s, 4 * i), U(s, 4 * i + 1));
  const double b = __dadd_rn(U(s, 4 * i + 2), U(s, 4 * i + 3));
  return __dmul_rn(__dsub_rn(__dadd_rn(a, b), 2.0), 1.7320508075688772);
}

// synth_embedding: per token t (seed s_t = hash_combine(seed,
// token)) raw_t[d] = fp32(N(s_t, d)), unit_t = Embedding(raw_t) (core.cpp:50-59:
// sequential fp64 sum of squares, inv = 1/sqrt, v*inv -> fp32); the prompt
// vector is Embedding(fp32(sum_t (double)unit_t[d])) with tokens summed in the
// given order. One thread per row; raw values are regenerated, not stored.
__global__ void k_synth_embeddings(const uint64_t* __restrict__ tok, const int32_t* __restrict__ n_tok, int max_tok,
                                   int64_t n, int dim, uint64_t seed, float* __restrict__ out, int* __restrict__ bad) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int nt = n_tok[r];
  if (nt < 1 || nt > max_tok) {
    atomicExch(bad, 1);
    return;
  }
  double inv[16];
  uint64_t st[16];
  for (int t = 0; t < nt && t < 16; ++t) {
    st[t] = hash_combine(seed, tok[r * max_tok + t]);
    double sq = 0.0;
    for (int d = 0; d < dim; ++d) {
      const float v = (float)N(st[t], d);
      sq = __fma_rn((double)v, (double)v, sq);
    }
    inv[t] = __ddiv_rn(1.0, __dsqrt_rn(sq));
  }
  float* o = out + r * dim;
  double sq = 0.0;
  for (int d = 0; d < dim; ++d) {
    double acc = 0.0;
    for (int t = 0; t < nt && t < 16; ++t) {
      const float v = (float)N(st[t], d);
      acc = __dadd_rn(acc, (double)(float)__dmul_rn((double)v, inv[t]));
    }
    const float fv = (float)acc;
    o[d] = fv;
    sq = __fma_rn((double)fv, (double)fv, sq);
  }
  const double iv = __ddiv_rn(1.0, __dsqrt_rn(sq));
  for (int d = 0; d < dim; ++d) o[d] = (float)__dmul_rn((double)o[d], iv);
}

// synth_latents per prompt seed p, S = 5 steps (5..25),
// F frames of E = H*W*C: stream seeds s(k) = hash_combine(p, k);
//   D[j][e]  = N(s(1), j*E + e)                 shared differential field
//   base[e]  = N(s(2), e)
//   first_i  = fp32(base*(1 - 0.05 i) + 0.05 N(s(3+i), e))
//   frame j of step i, j >= 1:
//     key:        fp32(first_i + alpha_i * D[j] * (1 + noise * N(s(10+i), j*E+e)))
//     redundant:  fp32(x_k + dup * N(s(20+i), j*E+e)), k a key of step i < j
//   frame 0 = first_i. Redundant sets nest across steps: the first
//   round(r_i (F-1)) entries of one permutation of 1..F-1 (Fisher-Yates with
//   ctr(s(30), t) % (t+1)); k = keys_so_far[ctr(s(40+i), j) % |keys_so_far|].
// The (frame -> source key) plan is built by one thread per (prompt, step);
// the elements are then independent (one thread each).
__global__ void k_synth_plan(const uint64_t* __restrict__ pseed, int64_t n, int F, const double* __restrict__ red,
                             int32_t* __restrict__ plan) {
  const int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (it >= n * 5) return;
  const int64_t p = it / 5;
  const int i = (int)(it % 5);
  const uint64_t s = pseed[p];
  int perm[256];
  for (int t = 0; t < F - 1; ++t) perm[t] = t + 1;
  for (int t = F - 2; t >= 1; --t) {
    const int q = (int)(hash_combine(hash_combine(s, 30), (uint64_t)t) % (uint64_t)(t + 1));
    const int x = perm[t];
    perm[t] = perm[q];
    perm[q] = x;
  }
  const int n_red = (int)floor(__dadd_rn(__dmul_rn(red[i], (double)(F - 1)), 0.5));
  bool is_red[256];
  for (int j = 0; j < F; ++j) is_red[j] = false;
  for (int t = 0; t < n_red && t < F - 1; ++t) is_red[perm[t]] = true;
  int keys[256];
  int nk = 1;
  keys[0] = 0;
  int32_t* pl = plan + it * F;
  pl[0] = -1;
  for (int j = 1; j < F; ++j) {
    if (is_red[j]) {
      pl[j] = keys[hash_combine(hash_combine(s, 40 + i), (uint64_t)j) % (uint64_t)nk];
    } else {
      pl[j] = -1;
      keys[nk++] = j;
    }
  }
}

struct LatentKnobs {
  double alpha[5];
  double noise, dup;
};

__device__ __forceinline__ float key_value(uint64_t s, int i, int j, int64_t e, int64_t E, const LatentKnobs& kn) {
  const double base = N(hash_combine(s, 2), (uint64_t)e);
  const double first =
      (double)(float)__dadd_rn(__dmul_rn(base, __dsub_rn(1.0, 0.05 * i)), __dmul_rn(0.05, N(hash_combine(s, 3 + i), (uint64_t)e)));
  if (j == 0) return (float)first;
  const double dj = N(hash_combine(s, 1), (uint64_t)(j * E + e));
  const double nz = __dadd_rn(1.0, __dmul_rn(kn.noise, N(hash_combine(s, 10 + i), (uint64_t)(j * E + e))));
  return (float)__dadd_rn(first, __dmul_rn(__dmul_rn(kn.alpha[i], dj), nz));
}

__global__ void k_synth_latents(const uint64_t* __restrict__ pseed, int64_t n, int F, int64_t E,
                                const int32_t* __restrict__ plan, LatentKnobs kn, float* __restrict__ out) {
  const int64_t total = n * 5 * F * E;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = x % E;
    const int64_t fr = x / E;  // (p, i, j)
    const int j = (int)(fr % F);
    const int64_t pi = fr / F;
    const int i = (int)(pi % 5);
    const uint64_t s = pseed[pi / 5];
    const int k = plan[pi * F + j];
    float v;
    if (k < 0) {
      v = key_value(s, i, j, e, E, kn);
    } else {
      const double xk = (double)key_value(s, i, k, e, E, kn);
      v = (float)__dadd_rn(xk, __dmul_rn(kn.dup, N(hash_combine(s, 20 + i), (uint64_t)(j * E + e))));
    }
    out[x] = v;
  }
}

// rectangular object masks drifting one pixel per frame,
// m = s(50): h0 = ctr(m,0) % (H/2), h1 = h0 + 1 + ctr(m,1) % (H - h0),
// w0 = ctr(m,2) % (W/2), w1 = w0 + 1 + ctr(m,3) % (W - w0); frame j shifts the
// rectangle by j % max(1, W - w1 + 1) columns; background = complement.
__global__ void k_synth_masks(const uint64_t* __restrict__ pseed, int64_t n, int F, int H, int W, int64_t mb,
                              uint8_t* __restrict__ om, uint8_t* __restrict__ bm) {
  const int64_t total = n * F * mb;
  for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < total; x += (int64_t)gridDim.x * blockDim.x) {
    const int64_t byte = x % mb;
    const int64_t pf = x / mb;
    const int j = (int)(pf % F);
    const uint64_t s = hash_combine(pseed[pf / F], 50);
    const int h0 = (int)(hash_combine(s, 0) % (uint64_t)(H / 2 > 0 ? H / 2 : 1));
    const int h1 = h0 + 1 + (int)(hash_combine(s, 1) % (uint64_t)(H - h0));
    const int w0 = (int)(hash_combine(s, 2) % (uint64_t)(W / 2 > 0 ? W / 2 : 1));
    const int w1 = w0 + 1 + (int)(hash_combine(s, 3) % (uint64_t)(W - w0));
    const int span = W - w1 + 1 > 1 ? W - w1 + 1 : 1;
    const int sh = j % span;
    uint8_t ob = 0, bb = 0;
    for (int b = 0; b < 8; ++b) {
      const int64_t px = byte * 8 + b;
      if (px >= (int64_t)H * W) break;
      const int y = (int)(px / W), xx = (int)(px % W);
      const bool in = y >= h0 && y < h1 && xx >= w0 + sh && xx < (w1 + sh < W ? w1 + sh : W);
      ob |= (uint8_t)(in ? 1 : 0) << b;
      bb |= (uint8_t)(in ? 0 : 1) << b;
    }
    om[x] = ob;
    bm[x] = bb;
  }
}

}  // namespace sg
}  // namespace fc

using namespace fc;

extern "C" {

lc_status lc_synth_embeddings(lc_ctx* ctx, const uint64_t* tokens, const int32_t* n_tokens, int max_tokens, int64_t n,
                              int dim, uint64_t seed, float* out) {
  LC_API_BEGIN
  FC_REQUIRE(ctx && tokens && n_tokens && out, "lc_synth_embeddings: null argument");
  FC_REQUIRE(dim > 0 && max_tokens >= 1 && max_tokens <= 16, "lc_synth_embeddings: dim > 0, 1..16 tokens per prompt");
  if (n <= 0) return LC_OK;
  DeviceGuard g(ctx->device);
  InArg<uint64_t> tk(ctx, tokens, (size_t)n * max_tokens);
  InArg<int32_t> nt(ctx, n_tokens, (size_t)n);
  OutArg<float> o(ctx, out, (size_t)n * dim);
  DevBuf bad(sizeof(int), ctx->stream);
  FC_CUDA(cudaMemsetAsync(bad.p, 0, sizeof(int), ctx->stream));
  sg::k_synth_embeddings<<<grid_for(n, 128), 128, 0, ctx->stream>>>(tk.dev, nt.dev, max_tokens, n, dim, seed, o.dev,
                                                                    bad.as<int>());
  FC_LAUNCH_CHECK();
  count_launch(ctx);
  o.finish(ctx);
  int hb = 0;
  FC_CUDA(cudaMemcpyAsync(&hb, bad.p, sizeof(int), cudaMemcpyDeviceToHost, ctx->stream));
  sync(ctx);
  if (hb) raise(LC_ERR_INVALID_ARGUMENT, "synth_embedding: token set must be nonempty (1..max_tokens)");
  LC_API_END
}

void lc_latent_spec_default(lc_latent_spec* s) {
  if (!s) return;
  const double r[5] = {0.9, 0.8, 0.6, 0.4, 0.25}, a[5] = {1.0, 0.9, 0.8, 0.7, 0.6};  // defaults.hpp:42-44
  for (int i = 0; i < 5; ++i) s->redundancy[i] = r[i], s->alpha[i] = a[i];
  s->noise_sigma = 0.01;
  s->dup_noise = 0.02;
}

lc_status lc_synth_latents(lc_ctx* ctx, const uint64_t* prompt_seeds, int64_t n, int F, int H, int W, int C,
                           const lc_latent_spec* spec, float* latents, uint8_t* obj_masks, uint8_t* bg_masks) {
  LC_API_BEGIN
  FC_REQUIRE(ctx && prompt_seeds && latents && obj_masks && bg_masks, "lc_synth_latents: null argument");
  FC_REQUIRE(F >= 1 && F <= 256 && H >= 1 && W >= 1 && C >= 1, "lc_synth_latents: bad geometry");
  lc_latent_spec sp;
  if (spec) sp = *spec;
  else lc_latent_spec_default(&sp);
  for (int i = 0; i < 5; ++i)
    FC_REQUIRE(sp.redundancy[i] >= 0.0 && sp.redundancy[i] <= 1.0, "LatentSpec: redundancy in [0, 1]");
  FC_REQUIRE(sp.noise_sigma >= 0.0 && sp.dup_noise >= 0.0, "LatentSpec: noise >= 0");
  if (n <= 0) return LC_OK;
  DeviceGuard g(ctx->device);
  const int64_t E = (int64_t)H * W * C, mb = ((int64_t)H * W + 7) / 8;
  InArg<uint64_t> ps(ctx, prompt_seeds, (size_t)n);
  OutArg<float> o(ctx, latents, (size_t)n * 5 * F * E);
  OutArg<uint8_t> om(ctx, obj_masks, (size_t)n * F * mb), bm(ctx, bg_masks, (size_t)n * F * mb);
  DevBuf red(5 * sizeof(double), ctx->stream), plan((size_t)n * 5 * F * sizeof(int32_t), ctx->stream);
  FC_CUDA(cudaMemcpyAsync(red.p, sp.redundancy, 5 * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  sg::k_synth_plan<<<grid_for(n * 5, 64), 64, 0, ctx->stream>>>(ps.dev, n, F, red.as<double>(), plan.as<int32_t>());
  sg::LatentKnobs kn;
  for (int i = 0; i < 5; ++i) kn.alpha[i] = sp.alpha[i];
  kn.noise = sp.noise_sigma;
  kn.dup = sp.dup_noise;
  sg::k_synth_latents<<<ctx->sm_count * 16, 256, 0, ctx->stream>>>(ps.dev, n, F, E, plan.as<int32_t>(), kn, o.dev);
  sg::k_synth_masks<<<grid_for(n * F * mb, 256, 1 << 16), 256, 0, ctx->stream>>>(ps.dev, n, F, H, W, mb, om.dev, bm.dev);
  FC_LAUNCH_CHECK();
  count_launch(ctx, 3);
  o.finish(ctx);
  om.finish(ctx);
  bm.finish(ctx);
  sync(ctx);
  LC_API_END
}

}  // extern "C"
