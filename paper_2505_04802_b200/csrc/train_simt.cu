// train_simt.cu -- the HBM-bound kernels of the training step:
// the Bayesian loss (readings R34 / R35), the stitch read backwards,
// LayerNorm backward, the attention backward's row statistics and the weight
// transposes the input-gradient GEMMs use.  The oracle is oracle/train.py.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "kernels.h"

namespace orbit2 {

namespace {

// inv_d = 1 / delta (hoisted: a multiply instead of two IEEE divisions per neighbour pair)
__device__ __forceinline__ float huber(float r, float delta, float inv_d) {
  const float a = fabsf(r);
  return a <= delta ? 0.5f * r * r * inv_d : a - 0.5f * delta;
}
__device__ __forceinline__ float huber_grad(float r, float delta, float inv_d) {
  return fabsf(r) <= delta ? r * inv_d : copysignf(1.f, r);
}

// Per output pixel i = (b, k, Y, X) of out [B][K][sH][sW]:
//   loss_b += ( w_Y (y - x)^2 + lambda sum_{j in C(i)} b_ij h(x_i - x_j) ) / n
//   dout    = ( -2 w_Y (y - x) + 2 lambda sum_j b_ij h'(x_i - x_j) ) / (n B)
// (C(i) symmetric and h' odd: the pairs (i, j) and (j, i) contribute equally to x_i.)
// Block = a 32 x 64 pixel tile of one (b, k) plane, staged with its 1-pixel ring in
// shared memory (coalesced row loads; every pixel read from HBM once); per-block sum
// in double, one atomicAdd per block.
constexpr int LT_Y = 32, LT_X = 64, LOSS_THREADS = 256;
__global__ void __launch_bounds__(LOSS_THREADS) loss_kernel(const float* __restrict__ out,
                                                            const float* __restrict__ truth, int B, int K, int sH,
                                                            int sW, float lam, float delta, int geo,
                                                            const float* __restrict__ latw, double* __restrict__ loss,
                                                            float* __restrict__ dout) {
  __shared__ float t[LT_Y + 2][LT_X + 2];
  const int plane = blockIdx.z;                 // b * K + k
  const int b = plane / K;
  const int Y0 = blockIdx.y * LT_Y, X0 = blockIdx.x * LT_X;
  const float* o = out + (int64_t)plane * sH * sW;
  for (int e = threadIdx.x; e < (LT_Y + 2) * (LT_X + 2); e += LOSS_THREADS) {
    const int ty = e / (LT_X + 2), tx = e - ty * (LT_X + 2);
    const int Y = Y0 + ty - 1, X = X0 + tx - 1;
    t[ty][tx] = (Y >= 0 && Y < sH && X >= 0 && X < sW) ? __ldg(o + (int64_t)Y * sW + X) : 0.f;
  }
  __syncthreads();
  const double n = (double)K * sH * sW;
  const float gscale = (float)(1.0 / (n * B));
  const float inv_d = 1.f / delta;
  double part = 0.0;
  const int tx = threadIdx.x & (LT_X - 1);
  for (int ty = threadIdx.x / LT_X; ty < LT_Y; ty += LOSS_THREADS / LT_X) {
    const int Y = Y0 + ty, X = X0 + tx;
    if (Y >= sH || X >= sW) continue;
    const float x = t[ty + 1][tx + 1];
    const int64_t gi = ((int64_t)plane * sH + Y) * sW + X;
    const float y = __ldg(truth + gi);
    const float w = geo ? __ldg(latw + Y) : 1.f;
    float tv = 0.f, g = 0.f;
#pragma unroll
    for (int dy = -1; dy <= 1; ++dy) {
#pragma unroll
      for (int dx = -1; dx <= 1; ++dx) {
        if (dy == 0 && dx == 0) continue;
        const int yy = Y + dy, xx = X + dx;
        if (yy < 0 || yy >= sH || xx < 0 || xx >= sW) continue;
        const float bij = (dy != 0 && dx != 0) ? 0.70710678118654752f : 1.f;
        const float r = x - t[ty + 1 + dy][tx + 1 + dx];
        tv += bij * huber(r, delta, inv_d);
        g += bij * huber_grad(r, delta, inv_d);
      }
    }
    const float dif = y - x;
    part += (double)(w * dif * dif + lam * tv);
    dout[gi] = (-2.f * w * dif + 2.f * lam * g) * gscale;
  }
  __shared__ double red[LOSS_THREADS / 32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) part += __shfl_xor_sync(0xffffffffu, part, off);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double sum = 0.0;
    for (int i = 0; i < LOSS_THREADS / 32; ++i) sum += red[i];
    atomicAdd(loss + b, sum / n);
  }
}

__global__ void lat_weights_kernel(float* w, int sH) {
  // w_r = cos(lat_r) / mean cos, lat_r = 90 - 180 (r + 1/2) / sH degrees (R35); one block
  __shared__ double sum;
  if (threadIdx.x == 0) sum = 0.0;
  __syncthreads();
  double loc = 0.0;
  for (int r = threadIdx.x; r < sH; r += blockDim.x) loc += cos((90.0 - 180.0 * (r + 0.5) / sH) * (M_PI / 180.0));
  atomicAdd(&sum, loc);
  __syncthreads();
  const double mean = sum / sH;
  for (int r = threadIdx.x; r < sH; r += blockDim.x)
    w[r] = (float)(cos((90.0 - 180.0 * (r + 0.5) / sH) * (M_PI / 180.0)) / mean);
}

// O6 read backwards: dG[b * chunk_core + t][(k P + al) P + be] = dout[b][k][P u + al][P w + be]
// for the chunk's output tokens t = (tile, u, w) (dec_hidden == 0: output = core tokens).
// One block per (token row, sample); threads over the K P^2 columns.
__global__ void stitch_bwd_kernel(const float* __restrict__ dout, __nv_bfloat16* __restrict__ dg, int64_t ldg,
                                  ChunkDev ch, int K, int P, int sH, int sW) {
  const int64_t t = blockIdx.x;   // output token within the chunk (one sample)
  const int b = blockIdx.y;
  __shared__ int s_tile;
  if (threadIdx.x == 0) {
    int lo = 0;
    for (int i = 1; i < ch.tc; ++i)
      if (ch.tiles[ch.tb + i].core_off - ch.core0 <= t) lo = i;
    s_tile = lo;
  }
  __syncthreads();
  const DevTile tl = ch.tiles[ch.tb + s_tile];
  const int64_t loc = t - (tl.core_off - ch.core0);
  const int u = tl.out_y0 + (int)(loc / tl.out_w), w = tl.out_x0 + (int)(loc % tl.out_w);
  const int Nh = K * P * P;
  __nv_bfloat16* row = dg + ((int64_t)b * ch.chunk_core + t) * ldg;
  for (int e = threadIdx.x; e < Nh; e += blockDim.x) {
    const int k = e / (P * P), ab = e - k * P * P, al = ab / P, be = ab - al * P;
    row[e] = __float2bfloat16_rn(
        __ldg(dout + (((int64_t)b * K + k) * sH + (int64_t)P * u + al) * sW + (int64_t)P * w + be));
  }
  for (int e = Nh + threadIdx.x; e < ldg; e += blockDim.x) row[e] = __float2bfloat16_rn(0.f);
}

// The same gather with 16-byte reads (P % 4 == 0, sW % 4 == 0): thread = (token, k, al, 4 be);
// SB_TPB tokens per block, each thread finds its token's tile by binary search over the
// (ascending) core offsets; writes of 4 bf16 (8 bytes) are contiguous along the dG row.
#ifndef ORBIT2_STITCH_BWD_VEC   // 0: the one-block-per-token kernel (A/B)
#define ORBIT2_STITCH_BWD_VEC 1
#endif
constexpr int SB_TPB = 16;
__global__ void stitch_bwd_vec_kernel(const float* __restrict__ dout, __nv_bfloat16* __restrict__ dg, int64_t ldg,
                                      ChunkDev ch, int K, int P, int sH, int sW) {
  const int b = blockIdx.y;
  const int q4 = P / 4, segs = K * P * q4;          // float4 segments per token
  const int64_t t0 = (int64_t)blockIdx.x * SB_TPB;
  const int Nh = K * P * P;
  for (int e = threadIdx.x; e < SB_TPB * segs; e += blockDim.x) {
    const int64_t t = t0 + e / segs;
    if (t >= ch.chunk_core) break;                   // e grows: every later e is past the end too
    const int sidx = e - (int)(e / segs) * segs;
    int lo = 0, hi = ch.tc - 1;                      // last tile with core_off - core0 <= t
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (ch.tiles[ch.tb + mid].core_off - ch.core0 <= t) lo = mid;
      else hi = mid - 1;
    }
    const DevTile& tl = ch.tiles[ch.tb + lo];
    const int64_t loc = t - (tl.core_off - ch.core0);
    const int u = tl.out_y0 + (int)(loc / tl.out_w), w = tl.out_x0 + (int)(loc % tl.out_w);
    const int k = sidx / (P * q4), rem = sidx - k * P * q4, al = rem / q4, q = rem - al * q4;
    const float4 v = __ldg(reinterpret_cast<const float4*>(
                               dout + (((int64_t)b * K + k) * sH + (int64_t)P * u + al) * sW + (int64_t)P * w) +
                           q);
    __nv_bfloat162 h2[2] = {__floats2bfloat162_rn(v.x, v.y), __floats2bfloat162_rn(v.z, v.w)};
    *reinterpret_cast<uint2*>(dg + ((int64_t)b * ch.chunk_core + t) * ldg + (k * P + al) * P + 4 * q) = *reinterpret_cast<const uint2*>(h2);
  }
  // zero the padding columns [Nh, ldg) of the block's tokens
  const int pad = (int)(ldg - Nh);
  for (int e = threadIdx.x; e < SB_TPB * pad; e += blockDim.x) {
    const int64_t t = t0 + e / pad;
    if (t >= ch.chunk_core) break;
    dg[((int64_t)b * ch.chunk_core + t) * ldg + Nh + (e - (int)(e / pad) * pad)] = __float2bfloat16_rn(0.f);
  }
}


// LayerNorm backward, one warp per row; lane l owns the float4 columns 4 l + 128 k
// (k < D / 128: coalesced 16-byte accesses):
//   xh = (z - mu) rstd;  dxh = dy g;  dz = rstd (dxh - mean(dxh) - xh mean(dxh xh))
// out = dres + dz (fp32) and a bf16 copy; dgamma += dy xh, dbeta += dy (per-lane partial
// sums, block reduction, atomics).  With a row map (LN_f over core rows): input row i
// reads z[zrow(i)] and writes dz there.
template <int P4>
__global__ void __launch_bounds__(256) ln_bwd_kernel(const float* __restrict__ dy, int64_t ldy,
                                                     const float* __restrict__ z, const float* __restrict__ g,
                                                     const float* __restrict__ dres, float* __restrict__ dz,
                                                     __nv_bfloat16* __restrict__ dz_bf, int64_t M, int D,
                                                     const int32_t* __restrict__ rowmap, int64_t map_per_b,
                                                     int64_t chunk_tokens, int64_t tok0,
                                                     float* __restrict__ dgamma, float* __restrict__ dbeta) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float4 ag[P4], ab[P4], gg[P4];
#pragma unroll
  for (int i = 0; i < P4; ++i) {
    ag[i] = ab[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    gg[i] = __ldg(reinterpret_cast<const float4*>(g) + lane + 32 * i);
  }
  const float invD = 1.f / D;
  for (int64_t row = (int64_t)blockIdx.x * 8 + warp; row < M; row += (int64_t)gridDim.x * 8) {
    int64_t zr = row;
    if (rowmap) {
      const int64_t b = row / map_per_b, rr = row - b * map_per_b;
      zr = b * chunk_tokens + (rowmap[rr] - tok0);
    }
    const float4* z4 = reinterpret_cast<const float4*>(z + zr * D);
    const float4* d4 = reinterpret_cast<const float4*>(dy + row * ldy);
    float4 zv[P4], dv[P4], rv[P4];
#pragma unroll
    for (int i = 0; i < P4; ++i) {
      zv[i] = __ldcs(z4 + lane + 32 * i);
      dv[i] = __ldcs(d4 + lane + 32 * i);
      rv[i] = dres ? __ldcs(reinterpret_cast<const float4*>(dres + zr * D) + lane + 32 * i)
                   : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < P4; ++i) s += (zv[i].x + zv[i].y) + (zv[i].z + zv[i].w);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mu = s * invD;
    float vs = 0.f;
#pragma unroll
    for (int i = 0; i < P4; ++i) {
      zv[i].x -= mu; zv[i].y -= mu; zv[i].z -= mu; zv[i].w -= mu;
      vs += zv[i].x * zv[i].x + zv[i].y * zv[i].y + zv[i].z * zv[i].z + zv[i].w * zv[i].w;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) vs += __shfl_xor_sync(0xffffffffu, vs, o);
    const float rstd = rsqrtf(vs * invD + 1e-5f);
    float m1 = 0.f, m2 = 0.f;
#pragma unroll
    for (int i = 0; i < P4; ++i) {
      float4 xh = make_float4(zv[i].x * rstd, zv[i].y * rstd, zv[i].z * rstd, zv[i].w * rstd);
      ag[i].x += dv[i].x * xh.x; ag[i].y += dv[i].y * xh.y; ag[i].z += dv[i].z * xh.z; ag[i].w += dv[i].w * xh.w;
      ab[i].x += dv[i].x; ab[i].y += dv[i].y; ab[i].z += dv[i].z; ab[i].w += dv[i].w;
      dv[i].x *= gg[i].x; dv[i].y *= gg[i].y; dv[i].z *= gg[i].z; dv[i].w *= gg[i].w;
      m1 += (dv[i].x + dv[i].y) + (dv[i].z + dv[i].w);
      m2 += dv[i].x * xh.x + dv[i].y * xh.y + dv[i].z * xh.z + dv[i].w * xh.w;
      zv[i] = xh;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      m1 += __shfl_xor_sync(0xffffffffu, m1, o);
      m2 += __shfl_xor_sync(0xffffffffu, m2, o);
    }
    m1 *= invD;
    m2 *= invD;
    float4* o4 = reinterpret_cast<float4*>(dz + zr * D);
    uint2* ob = reinterpret_cast<uint2*>(dz_bf + zr * D);
#pragma unroll
    for (int i = 0; i < P4; ++i) {
      float4 r;
      r.x = rv[i].x + rstd * (dv[i].x - m1 - zv[i].x * m2);
      r.y = rv[i].y + rstd * (dv[i].y - m1 - zv[i].y * m2);
      r.z = rv[i].z + rstd * (dv[i].z - m1 - zv[i].z * m2);
      r.w = rv[i].w + rstd * (dv[i].w - m1 - zv[i].w * m2);
      o4[lane + 32 * i] = r;
      __nv_bfloat162 lo = __floats2bfloat162_rn(r.x, r.y), hi = __floats2bfloat162_rn(r.z, r.w);
      ob[lane + 32 * i] = make_uint2(*reinterpret_cast<uint32_t*>(&lo), *reinterpret_cast<uint32_t*>(&hi));
    }
  }
  __shared__ float4 red[8][P4 * 32];   // block column sums: dgamma, then dbeta
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
#pragma unroll
    for (int i = 0; i < P4; ++i) red[warp][lane + 32 * i] = pass ? ab[i] : ag[i];
    __syncthreads();
    for (int c4 = threadIdx.x; c4 < D / 4; c4 += blockDim.x) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      for (int w = 0; w < 8; ++w) {
        const float4 t = red[w][c4];
        a.x += t.x; a.y += t.y; a.z += t.z; a.w += t.w;
      }
      float* dst = (pass ? dbeta : dgamma) + 4 * c4;
      atomicAdd(dst, a.x); atomicAdd(dst + 1, a.y); atomicAdd(dst + 2, a.z); atomicAdd(dst + 3, a.w);
    }
    __syncthreads();
  }
}

// Delta[h][row] = sum_{d < dh} dO[row][h dh + d] O[row][h dh + d]  (fp32), one thread per (row, head)
__global__ void delta_kernel(const __nv_bfloat16* __restrict__ dO, const __nv_bfloat16* __restrict__ O,
                             float* __restrict__ delta, int64_t M, int D, int heads, int64_t ld_stat) {
  // thread = one 16-byte chunk (8 values) of a row; the dh / 8 consecutive lanes of a head
  // (4, 8 or 16: a power of two dividing 32) reduce by shuffles, so a warp reads 512
  // contiguous bytes of dO and of O per step
  const int dh = D / heads, cph = dh / 8, cpr = D / 8;
  const int64_t n = M * cpr, n_pad = (n + 31) / 32 * 32;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_pad; e += (int64_t)gridDim.x * blockDim.x) {
    float s = 0.f;
    const bool valid = e < n;
    const int64_t row = valid ? e / cpr : 0;
    const int c = valid ? (int)(e - row * cpr) : 0;
    if (valid) {
      const uint4 x = __ldg(reinterpret_cast<const uint4*>(dO + row * D) + c);
      const uint4 y = __ldg(reinterpret_cast<const uint4*>(O + row * D) + c);
      const __nv_bfloat162* xp = reinterpret_cast<const __nv_bfloat162*>(&x);
      const __nv_bfloat162* yp = reinterpret_cast<const __nv_bfloat162*>(&y);
      float s2[2] = {0.f, 0.f};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float2 xf = __bfloat1622float2(xp[u]), yf = __bfloat1622float2(yp[u]);
        s2[u & 1] = fmaf(xf.x, yf.x, fmaf(xf.y, yf.y, s2[u & 1]));
      }
      s = s2[0] + s2[1];
    }
    for (int o = cph / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (valid && c % cph == 0) delta[(int64_t)(c / cph) * ld_stat + row] = s;
  }
}

// dqkv[row][0:D] = bf16(dq_acc[row][0:D])   (the Q columns; K / V written by the backward kernel)
__global__ void dq_convert_kernel(const float* __restrict__ dq, __nv_bfloat16* __restrict__ dqkv, int64_t M, int D) {
  const int64_t n4 = M * D / 4;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n4; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = (e * 4) / D, c = e * 4 - row * D;
    const float4 v = __ldg(reinterpret_cast<const float4*>(dq) + e);
    __nv_bfloat162* d = reinterpret_cast<__nv_bfloat162*>(dqkv + row * 3 * D + c);
    d[0] = __floats2bfloat162_rn(v.x, v.y);
    d[1] = __floats2bfloat162_rn(v.z, v.w);
  }
}

// W [n][k] fp32 (canonical, row-major) -> W^T [k][ld] bf16 (32 x 32 tiles through smem)
__global__ void transpose_bf16_kernel(const float* __restrict__ W, int n, int k, __nv_bfloat16* __restrict__ Wt,
                                      int64_t ld) {
  __shared__ float t[32][33];
  const int n0 = blockIdx.y * 32, k0 = blockIdx.x * 32;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int nn = n0 + i, kk = k0 + threadIdx.x;
    t[i][threadIdx.x] = (nn < n && kk < k) ? W[(int64_t)nn * k + kk] : 0.f;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int kk = k0 + i, nn = n0 + threadIdx.x;
    if (kk < k && nn < ld) Wt[(int64_t)kk * ld + nn] = __float2bfloat16_rn(nn < n ? t[threadIdx.x][i] : 0.f);
  }
}

// AdamW (R43): m = b1 m + (1 - b1) g; v = b2 v + (1 - b2) g^2;
// w -= lr (wd w + (m c1) / (sqrt(v c2) + eps)), c1 = 1 / (1 - b1^t), c2 = 1 / (1 - b2^t)
__global__ void adamw_kernel(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                             float* __restrict__ v, int64_t n, float lr, float b1, float b2, float eps, float wd,
                             float c1, float c2) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = fmaf(b1, m[i], (1.f - b1) * gi);
    const float vi = fmaf(b2, v[i], (1.f - b2) * gi * gi);
    m[i] = mi;
    v[i] = vi;
    const float wi = w[i];
    w[i] = wi - lr * fmaf(wd, wi, (mi * c1) / (sqrtf(vi * c2) + eps));
  }
}

}  // namespace

void launch_adamw(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2, float eps,
                  float wd, float c1, float c2, cudaStream_t st) {
  if (n <= 0) return;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 16LL * num_sms());
  adamw_kernel<<<blocks, 256, 0, st>>>(w, g, m, v, n, lr, b1, b2, eps, wd, c1, c2);
}

void launch_lat_weights(float* w, int sH, cudaStream_t st) { lat_weights_kernel<<<1, 256, 0, st>>>(w, sH); }

void launch_loss(const float* out, const float* truth, int B, int K, int sH, int sW, float lam, float delta, int geo,
                 const float* latw, double* loss, float* dout, cudaStream_t st) {
  dim3 grid((unsigned)((sW + LT_X - 1) / LT_X), (unsigned)((sH + LT_Y - 1) / LT_Y), (unsigned)(B * K));
  loss_kernel<<<grid, LOSS_THREADS, 0, st>>>(out, truth, B, K, sH, sW, lam, delta, geo, latw, loss, dout);
}

void launch_stitch_bwd(const float* dout, __nv_bfloat16* dg, int64_t ldg, const ChunkDev& ch, int B, int K, int P,
                       int sH, int sW, cudaStream_t st) {
  if (ch.chunk_core <= 0) return;
  if (P % 4 == 0 && sW % 4 == 0 && ldg % 4 == 0 && ORBIT2_STITCH_BWD_VEC) {
    const unsigned blocks = (unsigned)((ch.chunk_core + SB_TPB - 1) / SB_TPB);
    stitch_bwd_vec_kernel<<<dim3(blocks, (unsigned)B), 256, 0, st>>>(dout, dg, ldg, ch, K, P, sH, sW);
    return;
  }
  stitch_bwd_kernel<<<dim3((unsigned)ch.chunk_core, (unsigned)B), 192, 0, st>>>(dout, dg, ldg, ch, K, P, sH, sW);
}

bool launch_ln_bwd(const float* dy, int64_t ldy, const float* z, const float* g, const float* dres, float* dz,
                   __nv_bfloat16* dz_bf, int64_t M, int D, const int32_t* rowmap, int64_t map_per_b,
                   int64_t chunk_tokens, int64_t tok0, float* dgamma, float* dbeta, cudaStream_t st) {
  if (M <= 0) return true;
  if (D % 128 || ldy % 4) return false;
  const int blocks = (int)std::min<int64_t>((M + 7) / 8, 32LL * num_sms());
#define LNB(P_)                                                                                                \
  ln_bwd_kernel<P_><<<blocks, 256, 0, st>>>(dy, ldy, z, g, dres, dz, dz_bf, M, D, rowmap, map_per_b, chunk_tokens, \
                                            tok0, dgamma, dbeta);                                              \
  return true
  switch (D / 128) {
    case 1: LNB(1);
    case 2: LNB(2);
    case 3: LNB(3);
    case 4: LNB(4);
    case 5: LNB(5);
    case 6: LNB(6);
    case 7: LNB(7);
    case 8: LNB(8);
  }
#undef LNB
  return false;
}

void launch_delta(const __nv_bfloat16* dO, const __nv_bfloat16* O, float* delta, int64_t M, int D, int heads,
                  int64_t ld_stat, cudaStream_t st) {
  const int64_t n = M * (D / 8);
  if (n <= 0) return;
  const int blocks = (int)std::min<int64_t>((n + 255) / 256, 16LL * num_sms());
  delta_kernel<<<blocks, 256, 0, st>>>(dO, O, delta, M, D, heads, ld_stat);
}

void launch_dq_convert(const float* dq, __nv_bfloat16* dqkv, int64_t M, int D, cudaStream_t st) {
  const int64_t n4 = M * D / 4;
  if (n4 <= 0) return;
  const int blocks = (int)std::min<int64_t>((n4 + 255) / 256, 16LL * num_sms());
  dq_convert_kernel<<<blocks, 256, 0, st>>>(dq, dqkv, M, D);
}

void launch_transpose_bf16(const float* W, int n, int k, __nv_bfloat16* Wt, int64_t ld, cudaStream_t st) {
  dim3 grid((unsigned)((k + 31) / 32), (unsigned)((ld + 31) / 32));
  transpose_bf16_kernel<<<grid, dim3(32, 8), 0, st>>>(W, n, k, Wt, ld);
}

}  // namespace orbit2
