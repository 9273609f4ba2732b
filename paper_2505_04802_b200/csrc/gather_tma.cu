// gather_tma.cu -- step (1) tile gather with TMA-staged halo loads (bf16 path,
// CLAMP halos, reading R4).
//
// P:530 "each tile is extended with a fixed-width halo"; the padded rectangle of a
// tile is read as coarse pixels and rearranged into token-major patch rows
//     a[token (u,w)][(v p + dy) p + dx] = x[b, v, p u + dy, p w + dx]   (R1, O2/O3)
// One CTA per (padded token row u of a tile, tile, sample).  The CTA's input is
// one 3-D box of x viewed as [B*V][H][W]: V planes x p image rows x (segment of the
// row's p*pad_w pixels), moved into shared memory by a single
// cp.async.bulk.tensor.3d (the TMA engine generates full-line requests; no
// per-thread address arithmetic on the load side).  Threads then read the box
// token-fastest (conflict-free 8-byte shared loads for p = 2) and store each
// token's patch row in 16-byte pieces.  Patch rows have ld = round_up(Din, 8)
// columns: the zero columns up to the GEMM's K = round_up(Din, 64) are not
// written -- the embedding GEMM's TMA zero-fills them (GemmOperand::cols).
// In CLAMP mode every padded rectangle lies inside the grid, so the boxes never
// leave it except for the right-hand rounding of the box width (zero-filled,
// never used).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

namespace {

template <int P_>   // P_ = 2: specialised (every shipped config); 0: runtime p
__global__ void __launch_bounds__(128) gather_tma_kernel(const __grid_constant__ CUtensorMap tx,
                                                         __nv_bfloat16* __restrict__ patches,
                                                         int2* __restrict__ rowinfo, ChunkDev ch, int V, int p_rt,
                                                         int din, int ld, int segw, int sw) {
  const int p = P_ ? P_ : p_rt;
  extern __shared__ __align__(128) uint8_t gsm[];
  // sw = box width (pixels) >= p * segw + 3: the box starts at the 16-byte aligned
  // column at or left of the segment (a TMA box must start on a 16-byte boundary
  // in its innermost dimension; measured: an unaligned start is an illegal
  // instruction), `xo` pixels before the segment's first one
  float* sin = reinterpret_cast<float*>(gsm);               // [V][p][sw]
  uint64_t* bar = reinterpret_cast<uint64_t*>(gsm + (((size_t)V * p * sw * 4 + 15) & ~(size_t)15));
  const DevTile t = ch.tiles[ch.tb + blockIdx.y];
  const int ur = blockIdx.x;
  if (ur >= t.pad_h) return;
  const int b = blockIdx.z;
  const int64_t row0 = (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0) + (int64_t)ur * t.pad_w;
  const int u = t.pad_y0 + ur;
  if (threadIdx.x == 0) {
    tc::prefetch_tmap(&tx);
    tc::mbar_init(bar, 1);
    tc::fence_barrier_init();
  }
  __syncthreads();
  const uint32_t box_bytes = (uint32_t)V * p * sw * 4;
  const int nch = ld / 8;                                    // 16-byte pieces of a patch row
  const int pp = p * p;
  uint32_t phase = 0;
  for (int w0 = 0; w0 < t.pad_w; w0 += segw) {
    const int nw = min(segw, t.pad_w - w0);
    const int xs = p * (t.pad_x0 + w0);
    const int xa = xs & ~3, xo = xs - xa;                    // xo in {0, 2} for p = 2
    if (threadIdx.x == 0) {
      tc::mbar_arrive_expect_tx(bar, box_bytes);
      tc::tma_load_3d(&tx, sin, bar, xa, p * u, b * V);
    }
    tc::mbar_wait(bar, phase);
    phase ^= 1;
    for (int idx = threadIdx.x; idx < nw * nch; idx += blockDim.x) {
      const int tw = idx % nw, c = idx / nw;                 // token fastest: conflict-free smem reads
      uint32_t o[4];
      if constexpr (P_ == 2) {
        // columns 8c..8c+7 = variables v = 2c, 2c+1, each (dy, dx) in 2 x 2
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int v = 2 * c + h;
          float2 r0 = make_float2(0.f, 0.f), r1 = r0;
          if (v < V) {
            r0 = *reinterpret_cast<const float2*>(sin + (v * 2 + 0) * sw + xo + tw * 2);
            r1 = *reinterpret_cast<const float2*>(sin + (v * 2 + 1) * sw + xo + tw * 2);
          }
          o[2 * h] = tc::pack_bf16(r0.x, r0.y);
          o[2 * h + 1] = tc::pack_bf16(r1.x, r1.y);
        }
      } else {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const int col = 8 * c + e;
          f[e] = 0.f;
          if (col < din) {
            const int v = col / pp, r = col - v * pp, dy = r / p, dx = r - dy * p;
            f[e] = sin[(v * p + dy) * sw + xo + tw * p + dx];
          }
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) o[e] = tc::pack_bf16(f[2 * e], f[2 * e + 1]);
      }
      *reinterpret_cast<uint4*>(patches + (row0 + w0 + tw) * ld + 8 * c) = make_uint4(o[0], o[1], o[2], o[3]);
    }
    __syncthreads();                                         // sin read before the next box lands
  }
  for (int wr = threadIdx.x; wr < t.pad_w; wr += blockDim.x) rowinfo[row0 + wr] = make_int2(u, t.pad_x0 + wr);
}

}  // namespace

bool launch_gather_tma(const float* x, __nv_bfloat16* patches, int2* rowinfo, const ChunkDev& ch, int B, int V,
                       int H, int W, int p, int din, int ld, int max_pad_h, int max_pad_w, cudaStream_t st) {
  if (ld % 8 != 0 || ld < din || V > 256 || p > 8 || (W * 4) % 16 != 0) return false;
  // segment of tokens per box: box width p * segw <= 256 pixels, a multiple of 4
  // (16-byte rows); as wide as the widest padded row when that fits
  // tokens per box: the box (p * segw + 3 pixels rounded up to 16 bytes, <= 256)
  // covers the widest padded row when that fits
  const int segw = std::min(max_pad_w, (256 - 3) / p);
  const int sw = (segw * p + 3 + 3) & ~3;
  if (segw < 1 || sw > 256) return false;
  const size_t smem = (((size_t)V * p * sw * 4 + 15) & ~(size_t)15) + 16;
  if (smem > 200 * 1024) return false;
  CUtensorMap tx;
  if (!make_tmap_f32_3d(&tx, x, W, H, (int64_t)B * V, sw, p, V)) return false;
  dim3 grid(max_pad_h, ch.tc, B);
  if (p == 2) {
    static std::atomic<uint64_t> done{0};
    if (!smem_attr_once(reinterpret_cast<const void*>(gather_tma_kernel<2>), 200 * 1024, &done)) return false;
    gather_tma_kernel<2><<<grid, 128, smem, st>>>(tx, patches, rowinfo, ch, V, p, din, ld, segw, sw);
  } else {
    static std::atomic<uint64_t> done{0};
    if (!smem_attr_once(reinterpret_cast<const void*>(gather_tma_kernel<0>), 200 * 1024, &done)) return false;
    gather_tma_kernel<0><<<grid, 128, smem, st>>>(tx, patches, rowinfo, ch, V, p, din, ld, segw, sw);
  }
  return true;
}

}  // namespace orbit2
