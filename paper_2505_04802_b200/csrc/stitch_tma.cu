// stitch_tma.cu -- steps (4)-(5): crop + stitch + bilinear residual, bf16 tile_out,
// P = s * p = 8 (C1, C2, C3, C5).
//
// P:532 "the halo regions are discarded, and the non-padded tile outputs are
// stitched together"; P:498 residual upsample (R12: bilinear, align_corners =
// False, edge clamp).  For core token (u, w) of a tile and output variable k:
//     out[b, k, P u + al, P w + be] = g[token][(k P + al) P + be] + up_k(P u + al, P w + be)
// One CTA per (core token row u of a tile, tile, sample) writes the K x P output
// rows of that token row:
//   * the decoder outputs of variable k for the row's core tokens -- a
//     [core_w][P*P] bf16 box of tile_out -- arrive by one TMA tensor load
//     (128-byte swizzle: conflict-free shared reads), double-buffered over k so
//     the load of k + 2 overlaps the stores of k;
//   * the residual is separable: the CTA first interpolates along X the (at most
//     P/s + 2) input rows its output rows read, once, into shared memory; each
//     output element then needs two shared loads and one lerp in Y (instead of
//     four global loads per element);
//   * each thread stores whole float4 pieces of the output rows (coalesced).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz);

namespace {

constexpr int kP = 8;                 // output pixels per patch side handled here
constexpr int kRowB = kP * kP * 2;    // bytes of one token's variable-k block (128: one SW128 row)

__global__ void __launch_bounds__(256) stitch_tma_kernel(const __grid_constant__ CUtensorMap tt,
                                                         const float* __restrict__ x, float* __restrict__ out,
                                                         ChunkDev ch, const int32_t* __restrict__ cmap, int V, int H,
                                                         int W, int K, int s, int boxr, int nx_max, int nr_max) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = sm_raw + ((1024u - (tc::smem_u32(sm_raw) & 1023u)) & 1023u);
  const int slab_bytes = (boxr * kRowB + 1023) & ~1023;
  uint8_t* slab = sm;                                                   // [2][boxr][128 B] (SW128)
  float* hx = reinterpret_cast<float*>(sm + 2 * slab_bytes);            // [nr_max][nx_max]
  uint64_t* bar = reinterpret_cast<uint64_t*>(hx + (size_t)nr_max * nx_max);
  const DevTile t = ch.tiles[ch.tb + blockIdx.y];
  const int ur = blockIdx.x;
  if (ur >= t.core_h) return;
  const int b = blockIdx.z;
  const int u = t.core_y0 + ur;
  const int X0 = t.core_x0 * kP, NX = t.core_w * kP, NX4 = NX / 4;
  const int64_t sH = (int64_t)s * H, sW = (int64_t)s * W;
  const int32_t trow0 = (int32_t)((int64_t)b * ch.chunk_core + (t.core_off - ch.core0) + (int64_t)ur * t.core_w);
  const float inv_s = 1.0f / (float)s;
  auto src_row = [&](int Y, float* l) {   // O7: y0 and lambda of output row Y
    const float sy = fmaxf(((float)Y + 0.5f) * inv_s - 0.5f, 0.f);
    const int y0 = min((int)sy, H - 1);
    *l = sy - (float)y0;
    return y0;
  };
  float dummy;
  const int ylo = src_row(u * kP, &dummy);
  const int yhi = min(src_row(u * kP + kP - 1, &dummy) + 1, H - 1);
  const int nr = yhi - ylo + 1;
  const uint32_t box_bytes = (uint32_t)boxr * kRowB;
  if (threadIdx.x == 0) {
    tc::prefetch_tmap(&tt);
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    tc::fence_barrier_init();
    for (int k = 0; k < min(K, 2); ++k) {
      tc::mbar_arrive_expect_tx(&bar[k], box_bytes);
      tc::tma_load_2d(&tt, slab + k * slab_bytes, &bar[k], k * kP * kP, trow0);
    }
  }
  __syncthreads();
  for (int k = 0; k < K; ++k) {
    // residual rows of variable k interpolated along X (once per CTA)
    const float* plane = x + ((int64_t)b * V + cmap[k]) * H * W;
    for (int i = threadIdx.x; i < nr * NX; i += blockDim.x) {
      const int r = i / NX, xr = i - r * NX;
      const float sx = fmaxf(((float)(X0 + xr) + 0.5f) * inv_s - 0.5f, 0.f);
      const int xa = min((int)sx, W - 1), xb = min(xa + 1, W - 1);
      const float lx = sx - (float)xa;
      const float* row = plane + (int64_t)(ylo + r) * W;
      hx[r * nx_max + xr] = (1.f - lx) * __ldg(row + xa) + lx * __ldg(row + xb);
    }
    __syncthreads();
    tc::mbar_wait(&bar[k & 1], (k >> 1) & 1);
    const uint8_t* sl = slab + (k & 1) * slab_bytes;
    for (int i = threadIdx.x; i < kP * NX4; i += blockDim.x) {
      const int al = i / NX4, xr = 4 * (i - al * NX4);
      const int Y = u * kP + al;
      float ly;
      const int y0 = src_row(Y, &ly), y1 = min(y0 + 1, H - 1);
      const int wr = xr / kP, be = xr - wr * kP;
      const int byte = (al * kP + be) * 2;                 // within the token's 128-byte row
      const int chunk = (byte >> 4) ^ (wr & 7);            // SWIZZLE_128B
      const uint2 raw = *reinterpret_cast<const uint2*>(sl + wr * kRowB + chunk * 16 + (byte & 15));
      const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
      const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
      const float4 h0 = *reinterpret_cast<const float4*>(hx + (y0 - ylo) * nx_max + xr);
      const float4 h1 = *reinterpret_cast<const float4*>(hx + (y1 - ylo) * nx_max + xr);
      float4 o;
      o.x = __low2float(lo) + ((1.f - ly) * h0.x + ly * h1.x);
      o.y = __high2float(lo) + ((1.f - ly) * h0.y + ly * h1.y);
      o.z = __low2float(hi) + ((1.f - ly) * h0.z + ly * h1.z);
      o.w = __high2float(hi) + ((1.f - ly) * h0.w + ly * h1.w);
      *reinterpret_cast<float4*>(out + (((int64_t)b * K + k) * sH + Y) * sW + X0 + xr) = o;
    }
    __syncthreads();                                        // slab (k & 1) and hx consumed
    if (threadIdx.x == 0 && k + 2 < K) {
      tc::mbar_arrive_expect_tx(&bar[k & 1], box_bytes);
      tc::tma_load_2d(&tt, slab + (k & 1) * slab_bytes, &bar[k & 1], (k + 2) * kP * kP, trow0);
    }
  }
}

}  // namespace

bool launch_stitch_tma(const __nv_bfloat16* tile_out, int64_t tile_out_rows, const float* x, float* out,
                       const ChunkDev& ch, const int32_t* cmap, int B, int V, int H, int W, int K, int s, int P,
                       int max_core_h, int max_core_w, cudaStream_t st) {
  if (P != kP || ((int64_t)s * W) % 4 != 0 || max_core_w > 256 || max_core_w < 1 || tile_out_rows < 1) return false;
  const int boxr = max_core_w;
  const int nx_max = max_core_w * kP;
  const int nr_max = kP / s + 3;
  const size_t slab_bytes = ((size_t)boxr * kRowB + 1023) & ~(size_t)1023;
  const size_t smem = 1024 + 2 * slab_bytes + (size_t)nr_max * nx_max * 4 + 16;
  if (smem > 200 * 1024) return false;
  CUtensorMap tt;   // tile_out [rows][K * P * P] bf16, box [boxr][P * P] (128 B rows, SW128)
  if (!make_tmap_bf16(&tt, tile_out, tile_out_rows, (int64_t)K * kP * kP, (int64_t)K * kP * kP, boxr, kP * kP,
                      CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  static std::atomic<uint64_t> done{0};
  if (!smem_attr_once(reinterpret_cast<const void*>(stitch_tma_kernel), 200 * 1024, &done)) return false;
  dim3 grid(max_core_h, ch.tc, B);
  stitch_tma_kernel<<<grid, 256, smem, st>>>(tt, x, out, ch, cmap, V, H, W, K, s, boxr, nx_max, nr_max);
  return true;
}

}  // namespace orbit2
