// kernels_simt.cu -- CUDA-core kernels of the TILES pass: tile gather (step 1),
// LayerNorm, stitch + bilinear residual (steps 4-5), one-time table/weight
// preparation, and the IEEE-fp32 GEMM / attention used by the FP32 path.
//
// The bf16 contractions run on tcgen05 (gemm_tc.cu, attn_tc.cu); the fp32
// SIMT GEMM/attention here are the 1e-4 parity path (no TF32) and make no
// performance claim.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdlib>

#include "kernels.h"

namespace orbit2 {

template <typename T> __device__ __forceinline__ T to_out(float v);
template <> __device__ __forceinline__ float to_out<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 to_out<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }
template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

__device__ __forceinline__ float gelu_erf(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

// ---------------------------------------------------------------------------
// Step (1) tile gather.  One CTA per (padded token row u of a tile, tile, b).
// x~[v,a,c] = x[b, v, clamp(p*u0+a), clamp(p*w0+c)]  (clamp acts in REPLICATE
// mode only, R4); token column (v*p+dy)*p+dx (R1).  Writes the patch matrix
// row and the token's global patch coordinates (u, w) for the embed epilogue.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void gather_kernel(const float* __restrict__ x, T* __restrict__ patches, int2* __restrict__ rowinfo,
                              ChunkDev ch, int V, int H, int W, int p, int din, int din_pad) {
  const DevTile t = ch.tiles[ch.tb + blockIdx.y];
  const int ur = blockIdx.x;
  if (ur >= t.pad_h) return;
  const int b = blockIdx.z;
  const int64_t row0 = (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0) + (int64_t)ur * t.pad_w;
  const int u = t.pad_y0 + ur;
  const int pp = p * p;
  const float* xb = x + (int64_t)b * V * H * W;
  const int total = t.pad_w * din_pad;
  for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
    const int wr = idx / din_pad, col = idx - wr * din_pad;
    float val = 0.f;
    if (col < din) {
      const int v = col / pp, r = col - v * pp, dy = r / p, dx = r - dy * p;
      const int yy = min(max(p * u + dy, 0), H - 1);
      const int xx = min(max(p * (t.pad_x0 + wr) + dx, 0), W - 1);
      val = __ldg(xb + ((int64_t)v * H + yy) * W + xx);
    }
    patches[(row0 + wr) * din_pad + col] = to_out<T>(val);
  }
  for (int wr = threadIdx.x; wr < t.pad_w; wr += blockDim.x) rowinfo[row0 + wr] = make_int2(u, t.pad_x0 + wr);
}

// Staged variant: one CTA per (padded token row, tile, b) walks the row in
// segments of GSEG tokens.  Input pixels are read row-contiguously (coalesced:
// for each (v, dy) the p * GSEG pixels of one image row), scattered into a
// shared-memory [token][din] block (row stride padded against bank conflicts),
// then written out as whole 16-byte pieces of patch rows.
constexpr int GSEG = 64;
template <typename T>
__global__ void __launch_bounds__(128) gather_staged_kernel(const float* __restrict__ x, T* __restrict__ patches,
                                                            int2* __restrict__ rowinfo, ChunkDev ch, int V, int H,
                                                            int W, int p, int din, int din_pad) {
  extern __shared__ __align__(16) uint8_t gsm[];
  T* sp = reinterpret_cast<T*>(gsm);
  const int ld = din_pad + 16 / (int)sizeof(T);   // +16 bytes per row
  const DevTile t = ch.tiles[ch.tb + blockIdx.y];
  const int ur = blockIdx.x;
  if (ur >= t.pad_h) return;
  const int b = blockIdx.z;
  const int64_t row0 = (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0) + (int64_t)ur * t.pad_w;
  const int u = t.pad_y0 + ur;
  const int pp = p * p;
  const float* xb = x + (int64_t)b * V * H * W;
  constexpr int VEC = 16 / sizeof(T);
  for (int w0 = 0; w0 < t.pad_w; w0 += GSEG) {
    const int nw = min(GSEG, t.pad_w - w0);
    const int npx = nw * p;                           // image columns of the segment
    const int xpix0 = p * (t.pad_x0 + w0);
    __syncthreads();                                   // previous segment's stores have read sp
    for (int xl = threadIdx.x; xl < npx; xl += blockDim.x) {   // thread = image column
      const int wr = xl / p, dx = xl - wr * p;
      const float* src = xb + min(max(xpix0 + xl, 0), W - 1);
      T* dst = sp + wr * ld + dx;
      for (int dy = 0; dy < p; ++dy) {
        const float* s0 = src + (int64_t)min(max(p * u + dy, 0), H - 1) * W;
        int v = 0;
        for (; v + 8 <= V; v += 8) {   // 8 independent loads in flight per thread
          float f[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) f[k] = __ldg(s0 + (int64_t)(v + k) * H * W);
#pragma unroll
          for (int k = 0; k < 8; ++k) dst[(v + k) * pp + dy * p] = to_out<T>(f[k]);
        }
        for (; v < V; ++v) dst[v * pp + dy * p] = to_out<T>(__ldg(s0 + (int64_t)v * H * W));
      }
    }
    for (int idx = threadIdx.x; idx < nw * (din_pad - din); idx += blockDim.x) {
      const int wr = idx / (din_pad - din), c = din + idx - wr * (din_pad - din);
      sp[wr * ld + c] = to_out<T>(0.f);
    }
    __syncthreads();
    const int nv = din_pad / VEC;
    for (int idx = threadIdx.x; idx < nw * nv; idx += blockDim.x) {
      const int wr = idx / nv, c = (idx - wr * nv) * VEC;
      *reinterpret_cast<uint4*>(patches + (row0 + w0 + wr) * din_pad + c) =
          *reinterpret_cast<const uint4*>(sp + wr * ld + c);
    }
  }
  for (int wr = threadIdx.x; wr < t.pad_w; wr += blockDim.x) rowinfo[row0 + wr] = make_int2(u, t.pad_x0 + wr);
}

template <typename T>
void launch_gather(const float* x, T* patches, int2* rowinfo, const ChunkDev& ch, int B, int V, int H, int W,
                   int p, int din, int din_pad, int max_pad_h, cudaStream_t st) {
  dim3 grid(max_pad_h, ch.tc, B);
  const size_t smem = (size_t)GSEG * (din_pad + 16 / sizeof(T)) * sizeof(T);
  if (din_pad % (16 / sizeof(T)) == 0 && smem <= 48 * 1024)
    gather_staged_kernel<T><<<grid, 128, smem, st>>>(x, patches, rowinfo, ch, V, H, W, p, din, din_pad);
  else
    gather_kernel<T><<<grid, 256, 0, st>>>(x, patches, rowinfo, ch, V, H, W, p, din, din_pad);
}
template void launch_gather<float>(const float*, float*, int2*, const ChunkDev&, int, int, int, int, int, int, int,
                                   int, cudaStream_t);
template void launch_gather<__nv_bfloat16>(const float*, __nv_bfloat16*, int2*, const ChunkDev&, int, int, int,
                                           int, int, int, int, int, cudaStream_t);

// ---------------------------------------------------------------------------
// LayerNorm (R9: biased variance, eps 1e-5, affine), fp32 statistics.
// One warp per row; optional compaction of core rows for the head (R16).
// ---------------------------------------------------------------------------
template <typename T>
__global__ void layernorm_kernel(const float* __restrict__ z, const float* __restrict__ g,
                                 const float* __restrict__ bta, T* __restrict__ out, int64_t M, int D,
                                 bool compact, ChunkDev ch) {
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= M) return;
  int64_t src = r;
  if (compact) {
    const int64_t b = r / ch.chunk_core, rr = r - b * ch.chunk_core;
    src = b * ch.chunk_tokens + (ch.core_row[ch.core0 + rr] - ch.tok0);
  }
  const float4* zr = reinterpret_cast<const float4*>(z + src * D);
  const int n4 = D / 4;
  float s = 0.f;
  for (int i = lane; i < n4; i += 32) {
    float4 v = zr[i];
    s += (v.x + v.y) + (v.z + v.w);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / D;
  float q = 0.f;
  for (int i = lane; i < n4; i += 32) {
    float4 v = zr[i];
    float a = v.x - mean, b2 = v.y - mean, c = v.z - mean, e = v.w - mean;
    q += (a * a + b2 * b2) + (c * c + e * e);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q / D + 1e-5f);
  T* orow = out + r * D;
  for (int i = lane; i < n4; i += 32) {
    float4 v = zr[i];
    float4 gg = reinterpret_cast<const float4*>(g)[i];
    float4 bb = reinterpret_cast<const float4*>(bta)[i];
    orow[4 * i + 0] = to_out<T>((v.x - mean) * rstd * gg.x + bb.x);
    orow[4 * i + 1] = to_out<T>((v.y - mean) * rstd * gg.y + bb.y);
    orow[4 * i + 2] = to_out<T>((v.z - mean) * rstd * gg.z + bb.z);
    orow[4 * i + 3] = to_out<T>((v.w - mean) * rstd * gg.w + bb.w);
  }
}

// Register-resident variant for D = 128 * NV4: the row is read from HBM once
// (NV4 float4 per lane, coalesced), statistics from registers, one write.
__device__ __forceinline__ void store4(float* o, float a, float b, float c, float d) {
  *reinterpret_cast<float4*>(o) = make_float4(a, b, c, d);
}
__device__ __forceinline__ void store4(__nv_bfloat16* o, float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b), hi = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(o) = u;
}

template <typename T, int NV4>
__global__ void layernorm_reg_kernel(const float* __restrict__ z, const float* __restrict__ g,
                                     const float* __restrict__ bta, T* __restrict__ out, int64_t M, bool compact,
                                     ChunkDev ch) {
  constexpr int D = 128 * NV4;
  const int64_t r = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x & 31;
  if (r >= M) return;
  int64_t src = r;
  if (compact) {
    const int64_t b = r / ch.chunk_core, rr = r - b * ch.chunk_core;
    src = b * ch.chunk_tokens + (ch.core_row[ch.core0 + rr] - ch.tok0);
  }
  const float4* zr = reinterpret_cast<const float4*>(z + src * D);
  float4 v[NV4];
#pragma unroll
  for (int k = 0; k < NV4; ++k) v[k] = __ldcs(zr + lane + 32 * k);
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < NV4; ++k) s += (v[k].x + v[k].y) + (v[k].z + v[k].w);
#pragma unroll
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s * (1.0f / D);
  float q = 0.f;
#pragma unroll
  for (int k = 0; k < NV4; ++k) {
    const float a = v[k].x - mean, b2 = v[k].y - mean, c = v[k].z - mean, e = v[k].w - mean;
    q += (a * a + b2 * b2) + (c * c + e * e);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
  const float rstd = rsqrtf(q * (1.0f / D) + 1e-5f);
  T* orow = out + r * D;
#pragma unroll
  for (int k = 0; k < NV4; ++k) {
    const int c4 = lane + 32 * k;
    const float4 gg = __ldg(reinterpret_cast<const float4*>(g) + c4);
    const float4 bb = __ldg(reinterpret_cast<const float4*>(bta) + c4);
    store4(orow + 4 * c4, (v[k].x - mean) * rstd * gg.x + bb.x, (v[k].y - mean) * rstd * gg.y + bb.y,
           (v[k].z - mean) * rstd * gg.z + bb.z, (v[k].w - mean) * rstd * gg.w + bb.w);
  }
}

template <typename T>
void launch_layernorm(const float* z, const float* g, const float* b, T* out, int64_t M, int D,
                      const ChunkDev* compact, cudaStream_t st) {
  const int rows_per_cta = 8;
  dim3 grid((unsigned)((M + rows_per_cta - 1) / rows_per_cta));
  ChunkDev ch{};
  if (compact) ch = *compact;
  const bool cp = compact != nullptr;
  switch (D) {
    case 256: layernorm_reg_kernel<T, 2><<<grid, 32 * rows_per_cta, 0, st>>>(z, g, b, out, M, cp, ch); return;
    case 512: layernorm_reg_kernel<T, 4><<<grid, 32 * rows_per_cta, 0, st>>>(z, g, b, out, M, cp, ch); return;
    case 1024: layernorm_reg_kernel<T, 8><<<grid, 32 * rows_per_cta, 0, st>>>(z, g, b, out, M, cp, ch); return;
    case 2048: layernorm_reg_kernel<T, 16><<<grid, 32 * rows_per_cta, 0, st>>>(z, g, b, out, M, cp, ch); return;
    default: layernorm_kernel<T><<<grid, 32 * rows_per_cta, 0, st>>>(z, g, b, out, M, D, cp, ch);
  }
}
template void launch_layernorm<float>(const float*, const float*, const float*, float*, int64_t, int,
                                      const ChunkDev*, cudaStream_t);
template void launch_layernorm<__nv_bfloat16>(const float*, const float*, const float*, __nv_bfloat16*, int64_t,
                                              int, const ChunkDev*, cudaStream_t);

// ---------------------------------------------------------------------------
// Steps (4)+(5): crop/stitch + bilinear residual.  One CTA per (output row Y
// of a tile's core, tile, b); threads run over (k, X) with X fastest so the
// fp32 output row segment is written coalesced.
//   out[b,k,Y,X] = tile_out[row(b,t,token(u,w))][(k*P+al)*P+be] + up_k(Y,X)
//   up: src = max((Y+0.5)/s - 0.5, 0), y0 = floor, y1 = min(y0+1, H-1) (R12)
// ---------------------------------------------------------------------------
template <typename T>
__global__ void stitch_kernel(const T* __restrict__ tile_out, const float* __restrict__ x, float* __restrict__ out,
                              ChunkDev ch, const int32_t* __restrict__ cmap, int V, int H, int W, int K, int s,
                              int P) {
  const DevTile t = ch.tiles[ch.tb + blockIdx.y];
  const int yr = blockIdx.x;
  if (yr >= t.core_h * P) return;
  const int b = blockIdx.z;
  const int Y = t.core_y0 * P + yr;
  const int ur = yr / P, al = yr - ur * P;
  const int X0 = t.core_x0 * P, NX = t.core_w * P;
  const int64_t sH = (int64_t)s * H, sW = (int64_t)s * W;
  const int64_t trow0 = (int64_t)b * ch.chunk_core + (t.core_off - ch.core0) + (int64_t)ur * t.core_w;
  const int Nh = K * P * P;
  const float inv_s = 1.0f / (float)s;
  const float sy = fmaxf(((float)Y + 0.5f) * inv_s - 0.5f, 0.f);
  const int y0 = min((int)sy, H - 1), y1 = min(y0 + 1, H - 1);
  const float ly = sy - (float)y0;
  for (int idx = threadIdx.x; idx < K * NX; idx += blockDim.x) {
    const int k = idx / NX, xr = idx - k * NX;
    const int X = X0 + xr;
    const int wr = xr / P, be = xr - wr * P;
    const float vit = to_f32<T>(tile_out[(trow0 + wr) * Nh + (k * P + al) * P + be]);
    const float sx = fmaxf(((float)X + 0.5f) * inv_s - 0.5f, 0.f);
    const int x0 = min((int)sx, W - 1), x1 = min(x0 + 1, W - 1);
    const float lx = sx - (float)x0;
    const float* pl = x + ((int64_t)b * V + cmap[k]) * H * W;
    const float a00 = __ldg(pl + (int64_t)y0 * W + x0), a01 = __ldg(pl + (int64_t)y0 * W + x1);
    const float a10 = __ldg(pl + (int64_t)y1 * W + x0), a11 = __ldg(pl + (int64_t)y1 * W + x1);
    const float up = (1.f - ly) * ((1.f - lx) * a00 + lx * a01) + ly * ((1.f - lx) * a10 + lx * a11);
    out[(((int64_t)b * K + k) * sH + Y) * sW + X] = vit + up;
  }
}

// Vectorised variant for P % 4 == 0 (every shipped configuration): one CTA per
// (token row ur of a tile's core, tile, b) writes the P x K output rows of that
// token row.  A thread owns 4 consecutive output columns X (one float4 store per
// (k, al), one 8-byte tile_out load: the 4 columns share a token and be..be+3);
// column interpolation weights are computed once per thread, row weights once per
// al, no integer division in the inner loops.  The token row's tile_out slab
// (core_w x K P^2 values) is re-read across (k, al) from L1.
template <typename T>
__global__ void __launch_bounds__(128) stitch4_kernel(const T* __restrict__ tile_out, const float* __restrict__ x,
                                                      float* __restrict__ out, ChunkDev ch,
                                                      const int32_t* __restrict__ cmap, int V, int H, int W, int K,
                                                      int s, int P) {
  const DevTile t = ch.tiles[ch.tb + blockIdx.y];
  const int ur = blockIdx.x;
  if (ur >= t.core_h) return;
  const int b = blockIdx.z;
  const int X0 = t.core_x0 * P, NX4 = t.core_w * P / 4;
  const int64_t sH = (int64_t)s * H, sW = (int64_t)s * W;
  const int64_t trow0 = (int64_t)b * ch.chunk_core + (t.core_off - ch.core0) + (int64_t)ur * t.core_w;
  const int Nh = K * P * P;
  const float inv_s = 1.0f / (float)s;
  for (int c4 = threadIdx.x; c4 < NX4; c4 += blockDim.x) {
    const int xr = 4 * c4;
    const int wr = xr / P, be = xr - wr * P;
    const int X = X0 + xr;
    int xa[4], xb[4];
    float lx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float sx = fmaxf(((float)(X + e) + 0.5f) * inv_s - 0.5f, 0.f);
      xa[e] = min((int)sx, W - 1);
      xb[e] = min(xa[e] + 1, W - 1);
      lx[e] = sx - (float)xa[e];
    }
    const T* trow = tile_out + (trow0 + wr) * Nh + be;
    for (int al = 0; al < P; ++al) {
      const int Y = t.core_y0 * P + ur * P + al;
      const float sy = fmaxf(((float)Y + 0.5f) * inv_s - 0.5f, 0.f);
      const int y0 = min((int)sy, H - 1), y1 = min(y0 + 1, H - 1);
      const float ly = sy - (float)y0;
      for (int k = 0; k < K; ++k) {
        float vit[4];
        const T* src = trow + (k * P + al) * P;
        if constexpr (sizeof(T) == 2) {
          const uint2 raw = *reinterpret_cast<const uint2*>(src);
          const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
          const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
          vit[0] = __low2float(lo); vit[1] = __high2float(lo);
          vit[2] = __low2float(hi); vit[3] = __high2float(hi);
        } else {
          const float4 v = *reinterpret_cast<const float4*>(src);
          vit[0] = v.x; vit[1] = v.y; vit[2] = v.z; vit[3] = v.w;
        }
        const float* pl = x + ((int64_t)b * V + cmap[k]) * H * W;
        const float* r0 = pl + (int64_t)y0 * W;
        const float* r1 = pl + (int64_t)y1 * W;
        float o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float a00 = __ldg(r0 + xa[e]), a01 = __ldg(r0 + xb[e]);
          const float a10 = __ldg(r1 + xa[e]), a11 = __ldg(r1 + xb[e]);
          const float up = (1.f - ly) * ((1.f - lx[e]) * a00 + lx[e] * a01) + ly * ((1.f - lx[e]) * a10 + lx[e] * a11);
          o[e] = vit[e] + up;
        }
        *reinterpret_cast<float4*>(out + (((int64_t)b * K + k) * sH + Y) * sW + X) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
  }
}

// Separable variant (every shipped configuration: P % 4 == 0, p = P / s <= 2): the
// P output rows of a token row read at most p + 2 = 4 input rows, so each thread
// interpolates its 4 columns along X on those rows ONCE per variable (8 loads per
// row) and the P output rows only lerp in Y from registers -- 32 loads per
// (thread, k) instead of 16 per output row (the 4-load-per-element form is
// issue-bound: ncu issue 68 % at 2.7 TB/s).
// ORBIT2_STITCH_PER_ELEMENT=1: the 4-loads-per-element stitch4_kernel (A/B runs)
static bool stitch_per_element() {
  static const bool v = [] {
    const char* e = std::getenv("ORBIT2_STITCH_PER_ELEMENT");
    return e && e[0] == '1';
  }();
  return v;
}

template <typename T>
__global__ void __launch_bounds__(128) stitch4s_kernel(const T* __restrict__ tile_out, const float* __restrict__ x,
                                                       float* __restrict__ out, ChunkDev ch,
                                                       const int32_t* __restrict__ cmap, int V, int H, int W, int K,
                                                       int s, int P) {
  constexpr int NR = 4;
  const DevTile t = ch.tiles[ch.tb + blockIdx.y];
  const int ur = blockIdx.x;
  if (ur >= t.core_h) return;
  const int b = blockIdx.z;
  const int X0 = t.core_x0 * P, NX4 = t.core_w * P / 4;
  const int64_t sH = (int64_t)s * H, sW = (int64_t)s * W;
  const int64_t trow0 = (int64_t)b * ch.chunk_core + (t.core_off - ch.core0) + (int64_t)ur * t.core_w;
  const int Nh = K * P * P;
  const float inv_s = 1.0f / (float)s;
  const int Yb = (t.core_y0 + ur) * P;
  const int ylo = min((int)fmaxf(((float)Yb + 0.5f) * inv_s - 0.5f, 0.f), H - 1);
  for (int c4 = threadIdx.x; c4 < NX4; c4 += blockDim.x) {
    const int xr = 4 * c4;
    const int wr = xr / P, be = xr - wr * P;
    const int X = X0 + xr;
    int xa[4], xb[4];
    float lx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float sx = fmaxf(((float)(X + e) + 0.5f) * inv_s - 0.5f, 0.f);
      xa[e] = min((int)sx, W - 1);
      xb[e] = min(xa[e] + 1, W - 1);
      lx[e] = sx - (float)xa[e];
    }
    const T* trow = tile_out + (trow0 + wr) * Nh + be;
    for (int k = 0; k < K; ++k) {
      const float* pl = x + ((int64_t)b * V + cmap[k]) * H * W;
      float hx[NR][4];
#pragma unroll
      for (int r = 0; r < NR; ++r) {
        const float* row = pl + (int64_t)min(ylo + r, H - 1) * W;
#pragma unroll
        for (int e = 0; e < 4; ++e) hx[r][e] = (1.f - lx[e]) * __ldg(row + xa[e]) + lx[e] * __ldg(row + xb[e]);
      }
      for (int al = 0; al < P; ++al) {
        const int Y = Yb + al;
        const float sy = fmaxf(((float)Y + 0.5f) * inv_s - 0.5f, 0.f);
        const int y0 = min((int)sy, H - 1), y1 = min(y0 + 1, H - 1);
        const float ly = sy - (float)y0;
        const int r0 = y0 - ylo, r1 = y1 - ylo;   // in [0, NR) since P / s <= 2
        float vit[4];
        const T* src = trow + (k * P + al) * P;
        if constexpr (sizeof(T) == 2) {
          const uint2 raw = *reinterpret_cast<const uint2*>(src);
          const __nv_bfloat162 lo = *reinterpret_cast<const __nv_bfloat162*>(&raw.x);
          const __nv_bfloat162 hi = *reinterpret_cast<const __nv_bfloat162*>(&raw.y);
          vit[0] = __low2float(lo); vit[1] = __high2float(lo);
          vit[2] = __low2float(hi); vit[3] = __high2float(hi);
        } else {
          const float4 v = *reinterpret_cast<const float4*>(src);
          vit[0] = v.x; vit[1] = v.y; vit[2] = v.z; vit[3] = v.w;
        }
        float o[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          // registers indexed by the (warp-uniform) row offsets: select, not local memory
          float h0 = hx[0][e], h1 = hx[1][e];
#pragma unroll
          for (int r = 1; r < NR; ++r) {
            if (r0 == r) h0 = hx[r][e];
            if (r1 == r) h1 = hx[r][e];
          }
          o[e] = vit[e] + ((1.f - ly) * h0 + ly * h1);
        }
        *reinterpret_cast<float4*>(out + (((int64_t)b * K + k) * sH + Y) * sW + X) = make_float4(o[0], o[1], o[2], o[3]);
      }
    }
  }
}

template <typename T>
void launch_stitch(const T* tile_out, const float* x, float* out, const ChunkDev& ch, const int32_t* cmap, int B,
                   int V, int H, int W, int K, int s, int P, int max_core_h, cudaStream_t st) {
  // float4 stores need X and sW multiples of 4 (X0 = core_x0 * P: P % 4 == 0 and
  // sW = s W = P (W / p) ...: checked explicitly)
  const bool vec = P % 4 == 0 && ((int64_t)s * W) % 4 == 0;
  if (vec) {
    dim3 grid(max_core_h, ch.tc, B);
    if (P / s <= 2 && !stitch_per_element())
      stitch4s_kernel<T><<<grid, 128, 0, st>>>(tile_out, x, out, ch, cmap, V, H, W, K, s, P);
    else
      stitch4_kernel<T><<<grid, 128, 0, st>>>(tile_out, x, out, ch, cmap, V, H, W, K, s, P);
  } else {
    dim3 grid(max_core_h * P, ch.tc, B);
    stitch_kernel<T><<<grid, 256, 0, st>>>(tile_out, x, out, ch, cmap, V, H, W, K, s, P);
  }
}
template void launch_stitch<float>(const float*, const float*, float*, const ChunkDev&, const int32_t*, int, int,
                                   int, int, int, int, int, int, cudaStream_t);
template void launch_stitch<__nv_bfloat16>(const __nv_bfloat16*, const float*, float*, const ChunkDev&,
                                           const int32_t*, int, int, int, int, int, int, int, int, cudaStream_t);

// ---------------------------------------------------------------------------
// Rank-to-rank transfers (halo exchange / input gather): pack the rectangles of
// a [B][V][H][W] field into a contiguous message (rect by rect, [B][V][rows][cols])
// or scatter a message back.  One CTA per (rectangle, b*V + v); coalesced rows.
// ---------------------------------------------------------------------------
__global__ void xfer_kernel(const DevRect* __restrict__ rects, int H, int W, const float* __restrict__ src,
                            float* __restrict__ dst, int pack) {
  const DevRect r = rects[blockIdx.x];
  const int bv = blockIdx.y;
  const int rows = r.y1 - r.y0, cols = r.x1 - r.x0;
  const int64_t msg = r.off + (int64_t)bv * rows * cols;
  const int64_t fld = ((int64_t)bv * H + r.y0) * W + r.x0;
  for (int idx = threadIdx.x; idx < rows * cols; idx += blockDim.x) {
    const int y = idx / cols, x = idx - y * cols;
    if (pack) dst[msg + idx] = __ldg(src + fld + (int64_t)y * W + x);
    else dst[fld + (int64_t)y * W + x] = __ldg(src + msg + idx);
  }
}

void launch_xfer(const DevRect* rects, int count, int B, int V, int H, int W, const float* src, float* dst, int pack,
                 cudaStream_t st) {
  if (count == 0) return;
  dim3 grid(count, B * V);
  xfer_kernel<<<grid, 256, 0, st>>>(rects, H, W, src, dst, pack);
}

// ---------------------------------------------------------------------------
// One-time tables: sincos position rows (R7), computed in fp64 then rounded.
// pos_u[r][m] = sin(u om_m), pos_u[r][Q+m] = cos(u om_m), u = r - h, Q = D/4.
// ---------------------------------------------------------------------------
__global__ void pos_table_kernel(float* tab, int rows, int h, int D) {
  const int Q = D / 4;
  const int64_t n = (int64_t)rows * Q;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(i / Q), m = (int)(i - (int64_t)r * Q);
    const double om = pow(10000.0, -(double)m / (double)Q);
    const double a = (double)(r - h) * om;
    tab[(int64_t)r * (D / 2) + m] = (float)sin(a);
    tab[(int64_t)r * (D / 2) + Q + m] = (float)cos(a);
  }
}

void launch_pos_tables(float* pos_u, float* pos_w, int Hp, int Wp, int h, int D, cudaStream_t st) {
  pos_table_kernel<<<64, 256, 0, st>>>(pos_u, Hp + 2 * h, h, D);
  pos_table_kernel<<<64, 256, 0, st>>>(pos_w, Wp + 2 * h, h, D);
}

// fp32 [rows][cols] -> bf16/fp32 [rows][ld_dst] (zero-padded columns)
__global__ void convert_rows_kernel(const float* __restrict__ src, void* dst, int64_t rows, int64_t cols,
                                    int64_t ld_dst, int to_bf16) {
  const int64_t n = rows * ld_dst;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / ld_dst, c = i - r * ld_dst;
    const float v = c < cols ? src[r * cols + c] : 0.f;
    if (to_bf16)
      reinterpret_cast<__nv_bfloat16*>(dst)[i] = __float2bfloat16_rn(v);
    else
      reinterpret_cast<float*>(dst)[i] = v;
  }
}

void launch_convert_rows(const float* src, void* dst, int64_t rows, int64_t cols, int64_t ld_dst, int to_bf16,
                         cudaStream_t st) {
  int64_t n = rows * ld_dst;
  int blocks = (int)std::min<int64_t>((n + 255) / 256, 4096);
  convert_rows_kernel<<<blocks, 256, 0, st>>>(src, dst, rows, cols, ld_dst, to_bf16);
}

__global__ void add_vec_kernel(const float* a, const float* b, float* o, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    o[i] = a[i] + b[i];
}
void launch_add_vec(const float* a, const float* b, float* out, int64_t n, cudaStream_t st) {
  add_vec_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, st>>>(a, b, out, n);
}

// ---------------------------------------------------------------------------
// FP32 path: SIMT GEMM  C = A[M,K] . B[N,K]^T  with the shared epilogues.
// 64x64 tile, BK 16, 256 threads, 4x4 outputs per thread, IEEE fp32 FMA.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void epi_store(int epi, const EpiParams& ep, int64_t m, int64_t n, float acc) {
  const float v = acc + ep.bias[n];
  if (epi == EPI_BIAS) {
    reinterpret_cast<float*>(ep.C)[m * ep.ldc + n] = v;
  } else if (epi == EPI_GELU) {
    reinterpret_cast<float*>(ep.C)[m * ep.ldc + n] = gelu_erf(v);
  } else if (epi == EPI_RESID) {
    float* z = reinterpret_cast<float*>(ep.C) + m * ep.ldc + n;
    *z = *z + v;
  } else {
    const int2 uw = ep.rowinfo[m];
    const float pe = n < ep.half ? ep.pos_u[(int64_t)(uw.x + ep.pos_off) * ep.half + n]
                                 : ep.pos_w[(int64_t)(uw.y + ep.pos_off) * ep.half + (n - ep.half)];
    reinterpret_cast<float*>(ep.C)[m * ep.ldc + n] = v + pe;
  }
}

__global__ void __launch_bounds__(256) sgemm_kernel(int epi, const float* __restrict__ A, int64_t lda,
                                                    const float* __restrict__ Bw, int64_t ldb, int64_t M, int64_t N,
                                                    int64_t K, EpiParams ep) {
  __shared__ float As[16][64 + 4];
  __shared__ float Bs[16][64 + 4];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < K; k0 += 16) {
    for (int i = tid; i < 64 * 16; i += 256) {
      const int r = i / 16, c = i % 16;
      const int64_t gm = m0 + r, gn = n0 + r, gk = k0 + c;
      As[c][r] = (gm < M && gk < K) ? A[gm * lda + gk] : 0.f;
      Bs[c][r] = (gn < N && gk < K) ? Bw[gn * ldb + gk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) epi_store(epi, ep, m, n, acc[i][j]);
    }
}

void launch_sgemm(int epi, const float* A, int64_t lda, const float* Bw, int64_t ldb, int64_t M, int64_t N,
                  int64_t K, const EpiParams& ep, cudaStream_t st) {
  dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64));
  sgemm_kernel<<<grid, 256, 0, st>>>(epi, A, lda, Bw, ldb, M, N, K, ep);
}

// ---------------------------------------------------------------------------
// FP32 path: per-tile attention ("self-attention is restricted within
// each tile").  One CTA per (query block of 128 rows of a tile, head, sample);
// one query per thread; online softmax in fp32 with expf; keys masked to the
// tile.  out[row, h*d:(h+1)*d] = softmax(q K^T / sqrt(d)) V.
// ---------------------------------------------------------------------------
template <int DH>
__global__ void __launch_bounds__(128) attention_f32_kernel(const float* __restrict__ qkv, float* __restrict__ out,
                                                            ChunkDev ch, int D) {
  constexpr int KB = 32;
  __shared__ float Ks[KB][DH];
  __shared__ float Vs[KB][DH];
  const int g = ch.qb0 + blockIdx.x;
  const int li = ch.qblk_tile[g];
  const DevTile t = ch.tiles[li];
  const int h = blockIdx.y, b = blockIdx.z;
  const int qi = (g - t.qb_off) * kQBlock + threadIdx.x;
  const int64_t base = (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0);
  const int64_t ld = 3LL * D;
  const bool active = qi < t.n_tokens;
  float q[DH], o[DH];
  const float scale = rsqrtf((float)DH);
#pragma unroll
  for (int j = 0; j < DH; ++j) {
    q[j] = active ? qkv[(base + qi) * ld + h * DH + j] * scale : 0.f;
    o[j] = 0.f;
  }
  float m = -INFINITY, l = 0.f;
  for (int k0 = 0; k0 < t.n_tokens; k0 += KB) {
    const int nk = min(KB, t.n_tokens - k0);
    for (int i = threadIdx.x; i < KB * DH; i += blockDim.x) {
      const int r = i / DH, c = i % DH;
      const bool ok = r < nk;
      Ks[r][c] = ok ? qkv[(base + k0 + r) * ld + D + h * DH + c] : 0.f;
      Vs[r][c] = ok ? qkv[(base + k0 + r) * ld + 2 * D + h * DH + c] : 0.f;
    }
    __syncthreads();
    for (int r = 0; r < nk; ++r) {
      float sc = 0.f;
#pragma unroll
      for (int j = 0; j < DH; ++j) sc = fmaf(q[j], Ks[r][j], sc);
      const float mn = fmaxf(m, sc);
      const float corr = expf(m - mn);
      const float pr = expf(sc - mn);
      l = l * corr + pr;
#pragma unroll
      for (int j = 0; j < DH; ++j) o[j] = fmaf(pr, Vs[r][j], o[j] * corr);
      m = mn;
    }
    __syncthreads();
  }
  if (active) {
    const float inv = 1.f / l;
#pragma unroll
    for (int j = 0; j < DH; ++j) out[(base + qi) * D + h * DH + j] = o[j] * inv;
  }
}

void launch_attention_f32(const float* qkv, float* out, const ChunkDev& ch, int B, int D, int heads, int d,
                          cudaStream_t st) {
  dim3 grid(ch.nqb, heads, B);
  if (d == 32) attention_f32_kernel<32><<<grid, 128, 0, st>>>(qkv, out, ch, D);
  else if (d == 64) attention_f32_kernel<64><<<grid, 128, 0, st>>>(qkv, out, ch, D);
  else attention_f32_kernel<128><<<grid, 128, 0, st>>>(qkv, out, ch, D);
}

}  // namespace orbit2
