// gram_sm100.cu — K5 on the tensor cores: per (prompt, step) item the F x F
// frame Gram matrix that select_keyframes needs (codec.cpp:146-163 via
// frame_similarity, core.cpp:101-119), plus the EXACT squared norms.
//
// The reference's similarities are sequential fp64 sums over E = H*W*C
// elements; reproducing them for all F^2/2 pairs costs F^2/2 * E fp64 FMAs
// (14.8 ms for config[2] with the exact kernel). Here the Gram is computed
// APPROXIMATELY on tcgen05 with a rigorous error bound, and select_keyframes
// (k_select_cert, codec.cu) uses the exact sequential fp64 value for the few
// pairs whose decision the bound cannot settle. Outputs:
//   G~[item][F][F]  fp64, |G~(j,k) - dot(j,k)| <= GRAM_REL * sum_i |x_ji x_ki|
//                   <= GRAM_REL * ||x_j|| ||x_k||  (Cauchy-Schwarz)
//   nrm[item][F]    fp64, G~(j,j): the same approximation of sum_i x_ji^2,
//                   |nrm - ||x_j||^2| <= GRAM_REL ||x_j||^2. Consumers that
//                   need the reference's exact sequential value (exact
//                   select pairs, exact K7 fallback) recompute it
//                   (k_exact_norms, codec.cu); the certified K7 sums its own.
//   fmx[item][F]    u32, max_i |x_ji| as fp32 bits: exact zero-frame and
//                   non-finite detection (>= 0x7F800000) and the range guard
//                   of the error model below (select takes the exact path for
//                   an item whose frames leave [2^-40, 2^56]).
// Error model (bf16x3): x = hi + lo + r with hi = x rounded to bf16 (round
// half away from zero, done on the integer bits: (u + 0x8000) & 0xFFFF0000),
// lo = x - hi exact in fp32 (|lo| <= 2^-8 |x|), lo rounded to nearest bf16
// (|r| <= 2^-8 |lo| <= 2^-16 |x|); the MMAs form hi*hi' + hi*lo' + lo*hi'
// (each product exact in fp32), dropping lo*lo' and the r terms:
// <= 3.1 * 2^-16 |x x'|. The operand is the Gram of one tile with itself, so
// lo*hi' = (hi*lo')^T: two MMAs per K step (HH = hi hi', HL = hi lo') and
// G~(j,k) = (HH + HL)(j,k) + HL(k,j), the transpose added by the consumer
// (GT). Accumulation: fp32 in TMEM over chunks of 256 elements (<= 256 *
// 2^-23 relative to the chunk's sum |x x'|, truncating adders assumed),
// HH chunk totals added in fp64, HL chunk totals in fp32 (|HL| <= 2^-8
// sum|x x'|, so <= nchunks 2^-32 relative, negligible). Products that underflow fp32
// add <= 3 E 2^-126 in all, < 2^-17 of the bound when every frame's max |x|
// is >= 2^-40; max |x| <= 2^56 keeps chunk sums finite. GRAM_REL = 1e-4
// covers the sum (8.6e-5). Per element the split is integer/FADD work plus
// half a bf16x2 pack: no fp64.
//
// Tiles: two items (2 x F <= 128 frames) form the M = N = 128 operand; the
// cross-item blocks of the 128x128 product are unused (tensor throughput is
// not the limit: the kernel streams each latent once, HBM-bound).
// Warp roles (320 threads): 0 TMA producer (fp32 boxes of 32 elements),
// 1 MMA issuer (elected lane), 2-9 workers: thread = half a frame row of
// each K unit (max |x| + hi/lo split into SWIZZLE_128B bf16 tiles), and the
// TMEM -> fp64 chunk accumulation of 32 Gram columns of that row one chunk
// behind.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "sm100_ptx.cuh"

namespace fc {
namespace gram {

using namespace sm100;

constexpr int GT = 320;       // threads
constexpr int KU = 64;        // elements per K unit (one bf16 SW128 row)
constexpr int XBOX = 128 * 128;  // one fp32 box region: 128 rows x 32 fp32 (128 B)
constexpr int XSTAGE = 2 * XBOX; // a K unit = two fp32 boxes
constexpr int BTILE = 128 * 128; // one bf16 tile: 128 rows x 64 bf16
constexpr int BSTAGE = 2 * BTILE;  // hi + lo
constexpr int NX = 4, NB = 2;
constexpr int PF = 8;          // K units prefetched into L2 ahead of the smem ring
constexpr int CHUNK = 4;      // K units per fp32 TMEM accumulation chunk (256 elements)

struct Params {
  int n_items, F, n_tiles;
  int64_t E;
  int n_units;          // E / KU
  double* G;            // [n_items][F][F]
  float* GT;            // [n_items][F][F] HL; G~(j,k) = G(j,k) + GT(k,j)
  double* nrm;          // [n_items][F] G~(j,j)
  uint32_t* fmx;        // [n_items][F] max |x| bits
  int* bad;             // set to 1 if any element is non-finite (Frame ctor rule, core.cpp:11-25)
};

__device__ __forceinline__ void tma_prefetch_3d(const CUtensorMap* map, int x, int y, int z) {
  asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(reinterpret_cast<uint64_t>(map)),
               "r"(x), "r"(y), "r"(z)
               : "memory");
}

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(bar)
      : "memory");
}

// 16-byte chunk c of row r in a 128-B-row SWIZZLE_128B tile
__device__ __forceinline__ uint32_t sw128(int r, int c) { return (uint32_t)(r * 128 + ((c ^ (r & 7)) << 4)); }

__device__ __forceinline__ void lds128(uint32_t a, uint32_t (&v)[4]) {
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(a));
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
// bf16 pair (x0 low, x1 high) of the round-half-away hi parts and of the
// rounded remainders; exact lo = x - hi in between
__device__ __forceinline__ void split2(uint32_t u0, uint32_t u1, uint32_t& hi2, uint32_t& lo2) {
  const uint32_t h0 = (u0 + 0x8000u) & 0xFFFF0000u, h1 = (u1 + 0x8000u) & 0xFFFF0000u;
  const float l0 = __uint_as_float(u0) - __uint_as_float(h0), l1 = __uint_as_float(u1) - __uint_as_float(h1);
  hi2 = __byte_perm(h0, h1, 0x7632);
  const __nv_bfloat162 l2 = __floats2bfloat162_rn(l0, l1);  // one F2FP (RN) for the pair
  lo2 = *reinterpret_cast<const uint32_t*>(&l2);
}

__global__ void __launch_bounds__(GT, 1) k_gram_tc(const __grid_constant__ CUtensorMap tmX, Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* xst = base;                    // [NX][2][128 rows][128 B] fp32
  uint8_t* bst = base + NX * XSTAGE;      // [NB][hi, lo][128 rows][128 B] bf16
  uint64_t* bars = reinterpret_cast<uint64_t*>(bst + NB * BSTAGE);
  uint64_t* xfull = bars;
  uint64_t* xempty = xfull + NX;
  uint64_t* bfull = xempty + NX;
  uint64_t* bempty = bfull + NB;
  uint64_t* afull = bempty + NB;
  uint64_t* aempty = afull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(aempty + 2);
  __shared__ uint32_t s_mx[2][128];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int F = p.F;
  const int nu = p.n_units;
  const int nchunk = (nu + CHUNK - 1) / CHUNK;

  for (int i = threadIdx.x; i < (NX * XSTAGE) / 16; i += GT) reinterpret_cast<uint4*>(xst)[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) {
    for (int s = 0; s < NX; ++s) {
      mbar_init(smem_u32(&xfull[s]), 1);
      mbar_init(smem_u32(&xempty[s]), 8);
    }
    for (int s = 0; s < NB; ++s) {
      mbar_init(smem_u32(&bfull[s]), 8);
      mbar_init(smem_u32(&bempty[s]), 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(smem_u32(&afull[b]), 1);
      mbar_init(smem_u32(&aempty[b]), 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // zero-fill visible to TMA / MMA
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
      uint32_t u = 0;
      for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
        const int ia = 2 * tile, ib = 2 * tile + 1;
        const bool has_b = ib < p.n_items;
        const uint32_t bytes = (has_b ? 4u : 2u) * (uint32_t)F * 128u;
        // Units are visited from a per-tile rotation: with every SM at the
        // same element offset, the concurrent 256-B row segments (rows 4E
        // bytes apart) share their low address bits and pile onto a few HBM
        // channels (ncu: per-channel DRAM activity 17-35 %). The Gram and
        // norm sums are order-independent within their error bounds.
        const int shift = (int)(((int64_t)tile * 97) % nu);
        for (int k = 0; k < nu; ++k, ++u) {
          const int s = u % NX;
          const int kk = k + shift < nu ? k + shift : k + shift - nu;
          // the smem ring holds only NX units; keep PF more in flight to L2
          for (int kq = (k == 0 ? 0 : k + PF - 1); kq < nu && kq < k + PF; ++kq) {
            const int kw = kq + shift < nu ? kq + shift : kq + shift - nu;
            tma_prefetch_3d(&tmX, kw * KU, 0, ia);
            tma_prefetch_3d(&tmX, kw * KU + 32, 0, ia);
            if (has_b) {
              tma_prefetch_3d(&tmX, kw * KU, 0, ib);
              tma_prefetch_3d(&tmX, kw * KU + 32, 0, ib);
            }
          }
          mbar_wait(smem_u32(&xempty[s]), ((u / NX) & 1) ^ 1);
          mbar_expect_tx(smem_u32(&xfull[s]), bytes);
          uint8_t* dst = xst + s * XSTAGE;
          for (int h = 0; h < 2; ++h) {
            tma_load_3d(smem_u32(dst + h * XBOX), &tmX, smem_u32(&xfull[s]), kk * KU + h * 32, 0, ia);
            if (has_b) tma_load_3d(smem_u32(dst + h * XBOX + 64 * 128), &tmX, smem_u32(&xfull[s]), kk * KU + h * 32, 0, ib);
          }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(128 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    const bool issuer = elect_one();
    uint32_t u = 0, ch = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x) {
      for (int c = 0; c < nchunk; ++c, ++ch) {
        const uint32_t ab = ch & 1;
        mbar_wait(smem_u32(&aempty[ab]), ((ch >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + ab * 256;  // HH at +0, HL at +128
        const int k1 = min(nu, (c + 1) * CHUNK);
        for (int k = c * CHUNK; k < k1; ++k, ++u) {
          const int s = u % NB;
          mbar_wait(smem_u32(&bfull[s]), (u / NB) & 1);
          tc_fence_after();
          if (issuer) {
            const uint64_t dh = smem_desc_sw128(smem_u32(bst + s * BSTAGE));
            const uint64_t dl = smem_desc_sw128(smem_u32(bst + s * BSTAGE + BTILE));
#pragma unroll
            for (int t = 0; t < 4; ++t) {  // K = 16 per MMA; +32 B per step inside the swizzled row
              const uint64_t o = 2 * t;
              const uint32_t acc = (k != c * CHUNK || t != 0) ? 1u : 0u;
              mma_ss(d, dh + o, dh + o, idesc, acc);        // HH = hi hi'
              mma_ss(d + 128, dh + o, dl + o, idesc, acc);  // HL = hi lo'; lo hi' = HL^T

            }
          }
          if (issuer) tc_commit(smem_u32(&bempty[s]));
          __syncwarp();
        }
        if (issuer) tc_commit(smem_u32(&afull[ab]));
        __syncwarp();
      }
    }
  } else {
    // ---------------- 8 worker warps: convert half-rows + TMEM epilogue ----------------
    // warp w may only touch TMEM lanes 32*(w%4)..+31, so its row quarter is
    // w%4; warps 2-5 take elements 0-31 of every K unit (fp32 box 0), warps
    // 6-9 elements 32-63 (box 1). The epilogue of chunk c runs after the
    // conversion of chunk c+1 (the MMA lags the converters by about a unit).
    const int quarter = warp & 3;
    const int h = (warp - 2) >> 2;
    const int r = quarter * 32 + lane;  // row of the 128-row operand = TMEM lane
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const int colb = (r >> 6) * 64 + h * 32;  // this thread's 32 Gram columns
    uint32_t u = 0, ch = 0;
    int par = 0;
    for (int tile = blockIdx.x; tile < p.n_tiles; tile += gridDim.x, par ^= 1) {
      const int item = 2 * tile + (r >> 6);
      const int row = r & 63;
      const bool real = row < F && item < p.n_items;
      uint32_t mx = 0;  // max |x| bits of this half row
      double acc[32];  // sum over chunks of HH(row, col), fp64
      float acc2[32];  // sum over chunks of HL(row, col), fp32 (|HL| <= 2^-8 sum|x x'|)
#pragma unroll
      for (int i = 0; i < 32; ++i) acc[i] = 0.0, acc2[i] = 0.f;
      auto epilogue = [&](uint32_t gch) {
        const uint32_t ab = gch & 1;
        mbar_wait(smem_u32(&afull[ab]), (gch >> 1) & 1);
        tc_fence_after();
        float v[32];
        tmem_ld32(tmem + lane_base + ab * 256 + colb, v);  // HH
#pragma unroll
        for (int i = 0; i < 32; ++i) acc[i] += (double)v[i];
        tmem_ld32(tmem + lane_base + ab * 256 + 128 + colb, v);  // HL
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(smem_u32(&aempty[ab]));
#pragma unroll
        for (int i = 0; i < 32; ++i) acc2[i] += v[i];
      };
      const uint32_t ch0 = ch;
      for (int k = 0; k < nu; ++k, ++u) {
        const int sx = u % NX, sb = u % NB;
        mbar_wait(smem_u32(&xfull[sx]), (u / NX) & 1);
        mbar_wait(smem_u32(&bempty[sb]), ((u / NB) & 1) ^ 1);
        const uint32_t xb = smem_u32(xst) + sx * XSTAGE + h * XBOX;
        const uint32_t hi = smem_u32(bst) + sb * BSTAGE;
        const uint32_t lo = hi + BTILE;
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // bf16 chunk 4h+c = elements 8c..8c+7 of this box
          uint32_t x0[4], x1[4];
          lds128(xb + sw128(r, 2 * c), x0);
          lds128(xb + sw128(r, 2 * c + 1), x1);
#pragma unroll
          for (int e = 0; e < 4; ++e) mx = max(mx, max(x0[e] & 0x7FFFFFFFu, x1[e] & 0x7FFFFFFFu));
          uint32_t h2[4], l2[4];
          split2(x0[0], x0[1], h2[0], l2[0]);
          split2(x0[2], x0[3], h2[1], l2[1]);
          split2(x1[0], x1[1], h2[2], l2[2]);
          split2(x1[2], x1[3], h2[3], l2[3]);
          sts128(hi + sw128(r, 4 * h + c), h2[0], h2[1], h2[2], h2[3]);
          sts128(lo + sw128(r, 4 * h + c), l2[0], l2[1], l2[2], l2[3]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor-core reads
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(smem_u32(&xempty[sx]));
          mbar_arrive(smem_u32(&bfull[sb]));
        }
        if ((k + 1) % CHUNK == 0 && k + 1 > CHUNK) epilogue(ch++);  // chunk k/CHUNK - 1
      }
      while (ch < ch0 + (uint32_t)nchunk) epilogue(ch++);
      // row max |x| = max of the two halves (smem, double-buffered by tile parity)
      if (h == 1) s_mx[par][r] = mx;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      if (real) {
        if (h == 0) {
          const uint32_t m = max(mx, s_mx[par][r]);
          p.fmx[(int64_t)item * F + row] = m;
          if (m >= 0x7F800000u) atomicExch(p.bad, 1);  // inf / NaN element
        }
        if (h == (row >> 5)) {  // this thread holds column `row`: the diagonal HH + 2 HL
          double dg = 0.0;
#pragma unroll
          for (int i = 0; i < 32; ++i)
            if (i == (row & 31)) dg = acc[i] + 2.0 * (double)acc2[i];
          p.nrm[(int64_t)item * F + row] = dg;
        }
        double* g = p.G + ((int64_t)item * F + row) * F + h * 32;
        float* gt = p.GT + ((int64_t)item * F + row) * F + h * 32;
#pragma unroll
        for (int i = 0; i < 32; ++i)
          if (h * 32 + i < F) g[i] = acc[i] + (double)acc2[i], gt[i] = acc2[i];
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace gram

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn_gram() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    FC_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) raise(LC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// true when the tensor-core Gram applies: F <= 64 (two items per 128-row
// tile), F % 8 == 0, E % 64 == 0 and 16-byte aligned latents.
bool gram_tc_supported(int F, int64_t E, const float* lat) {
  const char* e = getenv("FC_GRAM_EXACT");
  if (e && atoi(e) == 1) return false;
  return F >= 8 && F <= 64 && F % 8 == 0 && E % 64 == 0 && E <= (int64_t)1 << 30 &&
         (reinterpret_cast<uintptr_t>(lat) & 15) == 0;
}

void gram_tc(lc_ctx* ctx, const float* lat, int n_items, int F, int64_t E, double* G, float* Gt, double* nrm,
             uint32_t* fmx, int* bad) {
  using namespace gram;
  alignas(64) CUtensorMap tm;
  cuuint64_t gdim[3] = {(cuuint64_t)E, (cuuint64_t)F, (cuuint64_t)n_items};
  cuuint64_t gstride[2] = {(cuuint64_t)E * 4, (cuuint64_t)F * E * 4};
  cuuint32_t box[3] = {32, (cuuint32_t)F, 1};
  cuuint32_t estride[3] = {1, 1, 1};
  CUresult r = encode_fn_gram()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(lat), gdim, gstride, box,
                                estride, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) raise(LC_ERR_CUDA, "cuTensorMapEncodeTiled (gram) failed: " + std::to_string((int)r));
  Params p;
  p.n_items = n_items;
  p.F = F;
  p.n_tiles = (n_items + 1) / 2;
  p.E = E;
  p.n_units = (int)(E / KU);
  p.G = G;
  p.GT = Gt;
  p.nrm = nrm;
  p.fmx = fmx;
  p.bad = bad;
  const size_t smem = 1024 + NX * XSTAGE + NB * BSTAGE + 256;
  FC_CUDA(cudaFuncSetAttribute(k_gram_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int grid = std::min(p.n_tiles, ctx->sm_count);
  KTimer kt(ctx, "gram");
  k_gram_tc<<<grid, GT, smem, ctx->stream>>>(tm, p);
  kt.stop();
  FC_LAUNCH_CHECK();
  count_launch(ctx);
}

}  // namespace fc
