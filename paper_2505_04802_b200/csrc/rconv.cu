// rconv.cu -- steps (4)-(5) with the optional convolutions of the Reslim decoder and
// residual path:
//   residual (reading R31):  res = up + conv_rb(GELU(conv_ra(up)))   [res_hidden > 0]
//                                   res = up                                 [otherwise]
//   decoder  (reading R32):  dec = conv_db(GELU(conv_da(vit)))       [dec_hidden > 0]
//                                   dec = vit                                [otherwise]
//   out = dec + res
// up = the bilinear x s upsample of the mapped input channels (O7); vit = the
// unpatchified linear-head output of the tile (tile_out), which with dec_hidden > 0
// covers the tile's core plus a ring of ceil(2/P) patches (the decoder's receptive
// field).  3x3 convolutions with bias, exact-erf GELU; zero padding outside the
// high-resolution field (residual) and outside the tile's output-token rectangle
// (decoder: at interior edges that zero band is never reached by a core pixel).
//
// One CTA per (block of P output rows x 64 columns of a tile's core, tile, sample):
// up (and vit) on the block grown by 2 pixels -> shared memory, the hidden layer on
// the block grown by 1 -> shared memory, the second convolution -> out.  fp32 FMA on
// the CUDA cores with the weights staged in shared memory.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <type_traits>

#include "kernels.h"

namespace orbit2 {

namespace {

constexpr int BX = 64;          // output columns per CTA
constexpr int RC_THREADS = 256;

template <typename T> __device__ __forceinline__ float ld_f32(const T* p);
template <> __device__ __forceinline__ float ld_f32<float>(const float* p) { return *p; }
template <> __device__ __forceinline__ float ld_f32<__nv_bfloat16>(const __nv_bfloat16* p) {
  return __bfloat162float(*p);
}

__device__ __forceinline__ float gelu_exact(float x) { return 0.5f * x * (1.0f + erff(x * 0.70710678118654752f)); }

// Weights are staged TRANSPOSED in shared memory, output channel fastest:
// wT[(i * 9 + dy * 3 + dx) * Cout + o] = W[o][i][dy][dx], so a thread that computes a
// group of 4 output channels of one pixel reads their 4 weights with one broadcast
// 16-byte shared load per input element (and the input element once per group).

// hidden = GELU(conv_a(src)) on the block grown by 1, zero where !inside(Y, X);
// thread = (pixel, group of 4 hidden channels)
template <typename Inside>
__device__ __forceinline__ void conv_hidden(const float* src, float* sh, const float* waT, const float* ba, int Cin,
                                            int C, int BY, int Y0, int X0, Inside inside) {
  const int UX = BX + 4, UY = BY + 4, HY = BY + 2, HX = BX + 2;
  const int C4 = C / 4, npx = HY * HX;
  for (int i = threadIdx.x; i < C4 * npx; i += RC_THREADS) {
    const int g = i / npx, r = i - g * npx, yy = r / HX, xx = r - yy * HX;
    float4 acc = make_float4(ba[4 * g], ba[4 * g + 1], ba[4 * g + 2], ba[4 * g + 3]);
    const bool in = inside(Y0 - 1 + yy, X0 - 1 + xx);
    if (in) {
      for (int k = 0; k < Cin; ++k) {
        const float* u = src + (k * UY + yy) * UX + xx;
        const float4* wk = reinterpret_cast<const float4*>(waT + (k * 9) * C) + g;
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
#pragma unroll
          for (int dx = 0; dx < 3; ++dx) {
            const float v = u[dy * UX + dx];
            const float4 wv = wk[(dy * 3 + dx) * C4];
            acc.x = fmaf(wv.x, v, acc.x); acc.y = fmaf(wv.y, v, acc.y);
            acc.z = fmaf(wv.z, v, acc.z); acc.w = fmaf(wv.w, v, acc.w);
          }
      }
    }
    float* h = sh + (4 * g * HY + yy) * HX + xx;
    h[0] = in ? gelu_exact(acc.x) : 0.f;
    h[HY * HX] = in ? gelu_exact(acc.y) : 0.f;
    h[2 * HY * HX] = in ? gelu_exact(acc.z) : 0.f;
    h[3 * HY * HX] = in ? gelu_exact(acc.w) : 0.f;
  }
}

// second convolution at output (k, al, xx) for k = 4 kg .. 4 kg + 3:
// b[k] + sum_c,dy,dx W[k][c][dy][dx] h[c][al+dy][xx+dx]   (K4 = padded K / 4)
__device__ __forceinline__ float4 conv_out4(const float* sh, const float* wbT, const float* bb, int C, int K4,
                                            int BY, int kg, int al, int xx) {
  const int HY = BY + 2, HX = BX + 2;
  float4 acc = make_float4(bb[4 * kg], bb[4 * kg + 1], bb[4 * kg + 2], bb[4 * kg + 3]);
  for (int c = 0; c < C; ++c) {
    const float* hp = sh + (c * HY + al) * HX + xx;
    const float4* wc = reinterpret_cast<const float4*>(wbT + (c * 9) * 4 * K4) + kg;
#pragma unroll
    for (int dy = 0; dy < 3; ++dy)
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const float v = hp[dy * HX + dx];
        const float4 wv = wc[(dy * 3 + dx) * K4];
        acc.x = fmaf(wv.x, v, acc.x); acc.y = fmaf(wv.y, v, acc.y);
        acc.z = fmaf(wv.z, v, acc.z); acc.w = fmaf(wv.w, v, acc.w);
      }
  }
  return acc;
}

// stage one conv pair transposed: W_a[C][K][3][3] b_a[C] W_b[K][C][3][3] b_b[K] ->
// waT[(k*9+t)*C + c], ba[C], wbT[(c*9+t)*K4p + k] (K padded to K4p = 4*ceil(K/4), zeros), bb[K4p]
__device__ __forceinline__ void stage_pair(const float* w, float* waT, float* ba, float* wbT, float* bb, int K, int C,
                                           int K4p) {
  for (int i = threadIdx.x; i < C * K * 9; i += RC_THREADS) {
    const int c = i / (K * 9), r = i - c * K * 9, k = r / 9, t = r - k * 9;
    waT[(k * 9 + t) * C + c] = w[i];
  }
  for (int i = threadIdx.x; i < C; i += RC_THREADS) ba[i] = w[C * K * 9 + i];
  const float* wb = w + C * K * 9 + C;
  for (int i = threadIdx.x; i < C * 9 * K4p; i += RC_THREADS) {
    const int ct = i / K4p, k = i - ct * K4p, c = ct / 9, t = ct - c * 9;
    wbT[i] = k < K ? wb[(k * C + c) * 9 + t] : 0.f;
  }
  for (int i = threadIdx.x; i < K4p; i += RC_THREADS) bb[i] = i < K ? wb[K * C * 9 + i] : 0.f;
}

// ORBIT2_CONV_MMA=1: the tensor-core form below for the bf16 path.  Measured slower
// than the FFMA form at C2 (res + dec hidden 8: 30.7 vs 13.0 ms per step; 16: 44.3 ms):
// the per-element im2col fragment loads (index arithmetic + scattered shared loads)
// cost more than the FFMAs they replace at these tiny channel counts.
#ifndef ORBIT2_CONV_MMA
#define ORBIT2_CONV_MMA 0
#endif
// ---- tensor-core form (bf16 path): the 3x3 convolution as an implicit GEMM on
// mma.sync.m16n8k16 (bf16 in, fp32 accumulate): rows = output pixels of an OY x OX
// grid, columns = output channels, K = Cin * 9 (im2col from the shared-memory input
// block of (OY + 2) x (OX + 2)).  The convolutions are 27-576 long per pixel, far
// below a tcgen05 tile, so the warp-level MMA is the right size.
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// weight fragments in mma order: frag[(s * NB + j) * 32 + lane] = (b0, b1) for k-step s, n-block j
__device__ __forceinline__ void stage_bfrag(const float* W, uint2* frag, int Cin, int Cout, int KS, int NB) {
  // W[o][ci][dy][dx] (PyTorch layout), B[kk][n] = W[n][kk] for kk < Cin * 9, n < Cout
  for (int i = threadIdx.x; i < KS * NB * 32; i += RC_THREADS) {
    const int lane = i & 31, sj = i >> 5, st = sj / NB, j = sj - st * NB;
    const int g = lane >> 2, tg = lane & 3, n = 8 * j + g;
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int kk = 16 * st + 2 * tg + (e & 1) + (e >> 1) * 8;
      v[e] = (n < Cout && kk < Cin * 9) ? W[(int64_t)n * Cin * 9 + kk] : 0.f;
    }
    frag[i] = make_uint2(pack_bf16x2(v[0], v[1]), pack_bf16x2(v[2], v[3]));
  }
}

// dst[n][y][x] = act(bias[n] + conv(src)[n][y][x]) for the OY x OX grid (0 where !inside)
template <bool GELU, typename Inside>
__device__ __forceinline__ void mma_conv(const float* src, int Cin, const uint2* frag, const float* bias, int Cout,
                                         int KS, int NB, int OY, int OX, float* dst, int dstX, Inside inside) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tg = lane & 3;
  const int SX = OX + 2, SY = OY + 2, npx = OY * OX, ntiles = (npx + 15) / 16;
  for (int tile = warp; tile < ntiles; tile += RC_THREADS / 32) {
    float acc[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
    int rowoff[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int m = min(tile * 16 + g + 8 * h, npx - 1);
      const int y = m / OX, x = m - y * OX;
      rowoff[h] = y * SX + x;
    }
    for (int st = 0; st < KS; ++st) {
      uint32_t a[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) {   // a0: (g, k), a1: (g+8, k), a2: (g, k+8), a3: (g+8, k+8); k = 2 tg, 2 tg + 1
        float v2[2];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int kk = 16 * st + 2 * tg + e + (r >> 1) * 8;
          float v = 0.f;
          if (kk < Cin * 9) {
            const int ci = kk / 9, t9 = kk - ci * 9, dy = t9 / 3, dx = t9 - dy * 3;
            v = src[ci * SY * SX + rowoff[r & 1] + dy * SX + dx];
          }
          v2[e] = v;
        }
        a[r] = pack_bf16x2(v2[0], v2[1]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (j >= NB) break;
        const uint2 b = frag[(st * NB + j) * 32 + lane];
        asm volatile(
            "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
            "{%0,%1,%2,%3};"
            : "+f"(acc[j][0]), "+f"(acc[j][1]), "+f"(acc[j][2]), "+f"(acc[j][3])
            : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b.x), "r"(b.y));
      }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j >= NB) break;
#pragma unroll
      for (int e = 0; e < 4; ++e) {   // c0, c1: row g; c2, c3: row g + 8; cols 2 tg, 2 tg + 1
        const int m = tile * 16 + g + 8 * (e >> 1), n = 8 * j + 2 * tg + (e & 1);
        if (m >= npx || n >= Cout) continue;
        const int y = m / OX, x = m - y * OX;
        float v = acc[j][e] + bias[n];
        if (GELU) v = inside(y, x) ? gelu_exact(v) : 0.f;
        dst[(n * OY + y) * dstX + x] = v;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(RC_THREADS) stitch_conv_kernel(
    const T* __restrict__ tile_out, const float* __restrict__ x, float* __restrict__ out, ChunkDev ch,
    const int32_t* __restrict__ cmap, const float* __restrict__ wres, const float* __restrict__ wdec, int V, int H,
    int W, int K, int s, int P, int CR, int CD, int nseg) {
  extern __shared__ __align__(16) float rsm[];
  const int BY = P;
  const int UY = BY + 4, UX = BX + 4;
  const int K4p = (K + 3) / 4 * 4;
  // staged pair sizes: waT C*K*9, ba C, wbT C*9*K4p, bb K4p
  const int nr = CR ? CR * K * 9 + CR + CR * 9 * K4p + K4p : 0, nd = CD ? CD * K * 9 + CD + CD * 9 * K4p + K4p : 0;
  float* sWr = rsm;                                 // [nr] residual conv pair, transposed
  float* sWd = sWr + nr;                            // [nd] decoder conv pair, transposed
  float* su = sWd + nd;                             // [K][UY][UX] up on the grown block
  float* sv = su + K * UY * UX;                     // [K][UY][UX] vit on the grown block (CD > 0)
  float* sh = sv + (CD ? K * UY * UX : 0);          // [max(CR, CD)][BY+2][BX+2] hidden layer
  float* sres = sh + max(CR, CD) * (BY + 2) * (BX + 2);   // [K][BY][BX] residual (CD > 0 && CR > 0)
  // tensor-core form (bf16 path): second-convolution results and the weight fragments
  constexpr bool MMA = ORBIT2_CONV_MMA && std::is_same<T, __nv_bfloat16>::value;
  const int KSa = (K * 9 + 15) / 16, NBo = (K + 7) / 8;
  const int KSr = (CR * 9 + 15) / 16, NBr = (CR + 7) / 8, KSd = (CD * 9 + 15) / 16, NBd = (CD + 7) / 8;
  float* scv = sres + (CD && CR ? K * BY * BX : 0);             // [K][BY][BX] conv_b + bias
  uint2* fra = reinterpret_cast<uint2*>(scv + (MMA ? K * BY * BX : 0));   // residual conv_a fragments
  uint2* frb = fra + (MMA && CR ? KSa * NBr * 32 : 0);                    // residual conv_b
  uint2* fda = frb + (MMA && CR ? KSr * NBo * 32 : 0);                    // decoder conv_a
  uint2* fdb = fda + (MMA && CD ? KSa * NBd * 32 : 0);                    // decoder conv_b
  const DevTile t = ch.tiles[ch.tb + blockIdx.y];
  const int ur = blockIdx.x / nseg, seg = blockIdx.x - ur * nseg;
  if (ur >= t.core_h || seg * BX >= t.core_w * P) return;
  const int b = blockIdx.z;
  const int Y0 = (t.core_y0 + ur) * P;
  const int X0 = t.core_x0 * P + seg * BX;
  const int nx = min(BX, t.core_w * P - seg * BX);
  const int sH = s * H, sW = s * W;
  const int tid = threadIdx.x;
  if (CR) stage_pair(wres, sWr, sWr + CR * K * 9, sWr + CR * K * 9 + CR, sWr + CR * K * 9 + CR + CR * 9 * K4p, K, CR, K4p);
  if (CD) stage_pair(wdec, sWd, sWd + CD * K * 9, sWd + CD * K * 9 + CD, sWd + CD * K * 9 + CD + CD * 9 * K4p, K, CD, K4p);
  if (MMA) {
    if (CR) {
      stage_bfrag(wres, fra, K, CR, KSa, NBr);
      stage_bfrag(wres + CR * K * 9 + CR, frb, CR, K, KSr, NBo);
    }
    if (CD) {
      stage_bfrag(wdec, fda, K, CD, KSa, NBd);
      stage_bfrag(wdec + CD * K * 9 + CD, fdb, CD, K, KSd, NBo);
    }
  }
  const float inv_s = 1.0f / (float)s;
  const int64_t tbase = (int64_t)b * ch.chunk_core + (t.core_off - ch.core0);   // tile's output tokens
  const int Nh = K * P * P;
  // up (and vit) on the block grown by 2
  for (int i = tid; i < K * UY * UX; i += RC_THREADS) {
    const int k = i / (UY * UX), r = i - k * UY * UX, yy = r / UX, xx = r - yy * UX;
    const int Y = Y0 - 2 + yy, X = X0 - 2 + xx;
    float v = 0.f;
    if (Y >= 0 && Y < sH && X >= 0 && X < sW) {
      const float sy = fmaxf(((float)Y + 0.5f) * inv_s - 0.5f, 0.f), sx = fmaxf(((float)X + 0.5f) * inv_s - 0.5f, 0.f);
      const int y0 = min((int)sy, H - 1), x0 = min((int)sx, W - 1);
      const int y1 = min(y0 + 1, H - 1), x1 = min(x0 + 1, W - 1);
      const float ly = sy - (float)y0, lx = sx - (float)x0;
      const float* pl = x + ((int64_t)b * V + cmap[k]) * H * W;
      const float a00 = __ldg(pl + (int64_t)y0 * W + x0), a01 = __ldg(pl + (int64_t)y0 * W + x1);
      const float a10 = __ldg(pl + (int64_t)y1 * W + x0), a11 = __ldg(pl + (int64_t)y1 * W + x1);
      v = (1.f - ly) * ((1.f - lx) * a00 + lx * a01) + ly * ((1.f - lx) * a10 + lx * a11);
    }
    su[i] = v;
    if (CD) {   // vit from the tile's output tokens; 0 outside the output-token rectangle
      const int u = Y >= 0 ? Y / P : -1, w = X >= 0 ? X / P : -1;
      float g = 0.f;
      if (u >= t.out_y0 && u < t.out_y0 + t.out_h && w >= t.out_x0 && w < t.out_x0 + t.out_w) {
        const int al = Y - u * P, be = X - w * P;
        g = ld_f32<T>(tile_out + (tbase + (int64_t)(u - t.out_y0) * t.out_w + (w - t.out_x0)) * Nh +
                      (k * P + al) * P + be);
      }
      sv[i] = g;
    }
  }
  __syncthreads();
  auto in_field = [&](int Y, int X) { return Y >= 0 && Y < sH && X >= 0 && X < sW; };
  const int K4 = K4p / 4, NP = BY * nx;
  auto in_field_h = [&](int yy, int xx) { return in_field(Y0 - 1 + yy, X0 - 1 + xx); };
  auto all_in = [](int, int) { return true; };
  if (CR) {   // residual path
    const float* wb = sWr + CR * K * 9 + CR;
    if (MMA) {
      mma_conv<true>(su, K, fra, sWr + CR * K * 9, CR, KSa, NBr, BY + 2, BX + 2, sh, BX + 2, in_field_h);
      __syncthreads();
      mma_conv<false>(sh, CR, frb, wb + CR * 9 * K4p, K, KSr, NBo, BY, BX, scv, BX, all_in);
    } else {
      conv_hidden(su, sh, sWr, sWr + CR * K * 9, K, CR, BY, Y0, X0, in_field);
    }
    __syncthreads();
    for (int i = tid; i < K4 * NP; i += RC_THREADS) {
      const int kg = i / NP, r = i - kg * NP, al = r / nx, xx = r - al * nx;
      float4 cv;
      if (MMA) {
        cv = make_float4(scv[((4 * kg) * BY + al) * BX + xx], 4 * kg + 1 < K ? scv[((4 * kg + 1) * BY + al) * BX + xx] : 0.f,
                         4 * kg + 2 < K ? scv[((4 * kg + 2) * BY + al) * BX + xx] : 0.f,
                         4 * kg + 3 < K ? scv[((4 * kg + 3) * BY + al) * BX + xx] : 0.f);
      } else {
        cv = conv_out4(sh, wb, wb + CR * 9 * K4p, CR, K4, BY, kg, al, xx);
      }
      const float cvs[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int k = 4 * kg + e;
        if (k >= K) break;
        const float res = su[(k * UY + al + 2) * UX + xx + 2] + cvs[e];
        if (CD) {
          sres[(k * BY + al) * BX + xx] = res;
        } else {   // decoder = the linear head: vit straight from tile_out
          const int xr = X0 - t.core_x0 * P + xx, wr = xr / P, be = xr - wr * P;
          const float vit = ld_f32<T>(tile_out + (tbase + (int64_t)ur * t.out_w + wr) * Nh + (k * P + al) * P + be);
          out[(((int64_t)b * K + k) * sH + Y0 + al) * sW + X0 + xx] = vit + res;
        }
      }
    }
    if (!CD) return;
    __syncthreads();   // sh is reused by the decoder
  }
  // decoder convolutions (CD > 0)
  const int oy0 = t.out_y0 * P, oy1 = (t.out_y0 + t.out_h) * P, ox0 = t.out_x0 * P, ox1 = (t.out_x0 + t.out_w) * P;
  auto in_out = [&](int Y, int X) { return Y >= oy0 && Y < oy1 && X >= ox0 && X < ox1; };
  const float* wb = sWd + CD * K * 9 + CD;
  if (MMA) {
    auto in_out_h = [&](int yy, int xx) { return in_out(Y0 - 1 + yy, X0 - 1 + xx); };
    mma_conv<true>(sv, K, fda, sWd + CD * K * 9, CD, KSa, NBd, BY + 2, BX + 2, sh, BX + 2, in_out_h);
    __syncthreads();
    mma_conv<false>(sh, CD, fdb, wb + CD * 9 * K4p, K, KSd, NBo, BY, BX, scv, BX, all_in);
  } else {
    conv_hidden(sv, sh, sWd, sWd + CD * K * 9, K, CD, BY, Y0, X0, in_out);
  }
  __syncthreads();
  for (int i = tid; i < K4 * NP; i += RC_THREADS) {
    const int kg = i / NP, r = i - kg * NP, al = r / nx, xx = r - al * nx;
    float4 dv;
    if (MMA) {
      dv = make_float4(scv[((4 * kg) * BY + al) * BX + xx], 4 * kg + 1 < K ? scv[((4 * kg + 1) * BY + al) * BX + xx] : 0.f,
                       4 * kg + 2 < K ? scv[((4 * kg + 2) * BY + al) * BX + xx] : 0.f,
                       4 * kg + 3 < K ? scv[((4 * kg + 3) * BY + al) * BX + xx] : 0.f);
    } else {
      dv = conv_out4(sh, wb, wb + CD * 9 * K4p, CD, K4, BY, kg, al, xx);
    }
    const float dvs[4] = {dv.x, dv.y, dv.z, dv.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int k = 4 * kg + e;
      if (k >= K) break;
      const float res = CR ? sres[(k * BY + al) * BX + xx] : su[(k * UY + al + 2) * UX + xx + 2];
      out[(((int64_t)b * K + k) * sH + Y0 + al) * sW + X0 + xx] = dvs[e] + res;
    }
  }
}

}  // namespace

template <typename T>
bool launch_stitch_conv(const T* tile_out, const float* x, float* out, const ChunkDev& ch, const int32_t* cmap,
                        const float* wres, const float* wdec, int B, int V, int H, int W, int K, int s, int P, int CR,
                        int CD, int max_core_h, int max_core_w, cudaStream_t st) {
  // hidden channels are computed 4 at a time (the planner accepts any 0..64; others are
  // rejected here, E_CUDA "launch configuration rejected")
  if (CR < 0 || CD < 0 || (CR == 0 && CD == 0) || CR % 4 || CD % 4) return false;
  const int nseg = (max_core_w * P + BX - 1) / BX;
  const size_t K4p = (size_t)(K + 3) / 4 * 4;
  const size_t nr = CR ? (size_t)CR * K * 9 + CR + (size_t)CR * 9 * K4p + K4p : 0;
  const size_t nd = CD ? (size_t)CD * K * 9 + CD + (size_t)CD * 9 * K4p + K4p : 0;
  const size_t up = (size_t)K * (P + 4) * (BX + 4);
  const bool mma = ORBIT2_CONV_MMA && std::is_same<T, __nv_bfloat16>::value;
  const size_t KSa = (K * 9 + 15) / 16, NBo = (K + 7) / 8;
  const size_t frags = !mma ? 0 : (CR ? KSa * ((CR + 7) / 8) * 32 + ((CR * 9 + 15) / 16) * NBo * 32 : 0) +
                                      (CD ? KSa * ((CD + 7) / 8) * 32 + ((CD * 9 + 15) / 16) * NBo * 32 : 0);
  const size_t smem = sizeof(float) * (nr + nd + up + (CD ? up : 0) + (size_t)std::max(CR, CD) * (P + 2) * (BX + 2) +
                                       (CD && CR ? (size_t)K * P * BX : 0) + (mma ? (size_t)K * P * BX : 0)) +
                      sizeof(uint2) * frags;
  if (smem > 200 * 1024) return false;
  static std::atomic<uint64_t> done{0};
  if (!smem_attr_once(reinterpret_cast<const void*>(stitch_conv_kernel<T>), 200 * 1024, &done)) return false;
  dim3 grid(max_core_h * nseg, ch.tc, B);
  stitch_conv_kernel<T><<<grid, RC_THREADS, smem, st>>>(tile_out, x, out, ch, cmap, wres, wdec, V, H, W, K, s, P, CR,
                                                        CD, nseg);
  return true;
}
template bool launch_stitch_conv<float>(const float*, const float*, float*, const ChunkDev&, const int32_t*,
                                        const float*, const float*, int, int, int, int, int, int, int, int, int, int,
                                        int, cudaStream_t);
template bool launch_stitch_conv<__nv_bfloat16>(const __nv_bfloat16*, const float*, float*, const ChunkDev&,
                                                const int32_t*, const float*, const float*, int, int, int, int, int,
                                                int, int, int, int, int, int, cudaStream_t);

}  // namespace orbit2
