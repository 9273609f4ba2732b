// compress.cu -- adaptive spatial compression (readings
// R37-R40; the oracle is oracle/compress.py).
//
//   partition : Canny edge map (blur, Sobel, non-maximum suppression, double threshold,
//               hysteresis) -> per max_side cell a quad-tree of edge densities -> leaves
//               compacted in (image, row, col) order
//   tokenize  : each leaf average-pooled to min_side^2 per channel, linear embedding + the
//               leaf level's scale embedding (one fp32 GEMM over all leaves)
//   detokenize: linear projection (one fp32 GEMM), nearest-neighbour broadcast over the
//               leaf, 3x3 smoothing
//
// The Canny decision is boolean, so its arithmetic is the oracle's: float32 with every
// product and sum rounded separately (__fmul_rn / __fadd_rn: no contraction into FMA),
// correctly rounded sqrt, the same summation order.  HBM-bound stencils: one thread per
// pixel, coalesced rows; hysteresis propagates inside 32 x 32 shared-memory tiles and
// repeats over the field until nothing changes (host loop on a device flag).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>

#include "kernels.h"

namespace orbit2 {

namespace {

constexpr int MAX_TAPS = 17;   // sigma <= 8/3 (radius ceil(3 sigma) <= 8)
struct Taps {
  float w[MAX_TAPS];
  int r;
};

__device__ __forceinline__ int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

// rows then columns (R37 order: taps i = -r .. r, acc = acc + w_i v)
__global__ void blur_h_kernel(const float* __restrict__ in, float* __restrict__ out, int H, int W, Taps t) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, b = blockIdx.z;
  if (x >= W) return;
  const float* row = in + ((int64_t)b * H + y) * W;
  float acc = 0.f;
  for (int i = -t.r; i <= t.r; ++i) acc = __fadd_rn(acc, __fmul_rn(t.w[i + t.r], __ldg(row + clampi(x + i, 0, W - 1))));
  out[((int64_t)b * H + y) * W + x] = acc;
}
__global__ void blur_v_kernel(const float* __restrict__ in, float* __restrict__ out, int H, int W, Taps t) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, b = blockIdx.z;
  if (x >= W) return;
  const float* img = in + (int64_t)b * H * W;
  float acc = 0.f;
  for (int i = -t.r; i <= t.r; ++i)
    acc = __fadd_rn(acc, __fmul_rn(t.w[i + t.r], __ldg(img + (int64_t)clampi(y + i, 0, H - 1) * W + x)));
  out[((int64_t)b * H + y) * W + x] = acc;
}

// Sobel (edge replication), magnitude, direction bin (0 horizontal, 1 vertical, 2 / 3
// diagonals), per-image max magnitude (float bits of a non-negative value order as ints)
__global__ void sobel_kernel(const float* __restrict__ bl, float* __restrict__ mag, uint8_t* __restrict__ dir, int H,
                             int W, unsigned* __restrict__ gmax) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, b = blockIdx.z;
  float m = 0.f;
  if (x < W) {
    const float* img = bl + (int64_t)b * H * W;
    auto p = [&](int dy, int dx) {
      return __ldg(img + (int64_t)clampi(y + dy, 0, H - 1) * W + clampi(x + dx, 0, W - 1));
    };
    const float right = __fadd_rn(__fadd_rn(p(-1, 1), __fmul_rn(2.f, p(0, 1))), p(1, 1));
    const float left = __fadd_rn(__fadd_rn(p(-1, -1), __fmul_rn(2.f, p(0, -1))), p(1, -1));
    const float down = __fadd_rn(__fadd_rn(p(1, -1), __fmul_rn(2.f, p(1, 0))), p(1, 1));
    const float up = __fadd_rn(__fadd_rn(p(-1, -1), __fmul_rn(2.f, p(-1, 0))), p(-1, 1));
    const float gx = __fsub_rn(right, left), gy = __fsub_rn(down, up);
    m = __fsqrt_rn(__fadd_rn(__fmul_rn(gx, gx), __fmul_rn(gy, gy)));
    const float ax = fabsf(gx), ay = fabsf(gy);
    const float t22 = 0.41421356237309503f;
    uint8_t d = __fmul_rn(gx, gy) > 0.f ? 2 : 3;
    if (__fmul_rn(t22, ay) >= ax) d = 1;
    if (__fmul_rn(t22, ax) >= ay) d = 0;
    const int64_t o = ((int64_t)b * H + y) * W + x;
    mag[o] = m;
    dir[o] = d;
  }
  // block max -> one atomic per block
  __shared__ float red[32];
  float v = m;
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, s));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) v = fmaxf(v, red[i]);
    v = fmaxf(v, red[0]);
    atomicMax(gmax + b, __float_as_uint(v));
  }
}

// NMS + double threshold: 2 = strong (>= high), 1 = weak (>= low), 0 otherwise
__global__ void nms_kernel(const float* __restrict__ mag, const uint8_t* __restrict__ dir, uint8_t* __restrict__ lab,
                           int H, int W, const unsigned* __restrict__ gmax, float low_frac, float high_frac) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y, b = blockIdx.z;
  if (x >= W) return;
  const float* mg = mag + (int64_t)b * H * W;
  const int64_t o = (int64_t)y * W + x;
  const float m = mg[o];
  const int d = dir[(int64_t)b * H * W + o];
  const int dy1 = d == 0 ? 0 : -1, dx1 = d == 0 ? -1 : (d == 1 ? 0 : (d == 2 ? -1 : 1));
  auto at = [&](int yy, int xx) { return (yy < 0 || yy >= H || xx < 0 || xx >= W) ? 0.f : mg[(int64_t)yy * W + xx]; };
  const float a = at(y + dy1, x + dx1), c = at(y - dy1, x - dx1);
  const float gm = __uint_as_float(gmax[b]);
  const float lo = __fmul_rn(low_frac, gm), hi = __fmul_rn(high_frac, gm);
  uint8_t l = 0;
  if (gm > 0.f && m > 0.f && m >= a && m >= c) l = m >= hi ? 2 : (m >= lo ? 1 : 0);
  lab[(int64_t)b * H * W + o] = l;
}

// Hysteresis: weak pixels 8-connected to strong ones become strong.  A 32 x 32 tile (+1 ring)
// in shared memory iterates to its local fixed point; *changed is raised when any pixel of
// the field changed (the host repeats until a pass changes nothing).
constexpr int HT = 32;
__global__ void __launch_bounds__(HT * 8) hyst_kernel(uint8_t* __restrict__ lab, int H, int W,
                                                      int* __restrict__ changed) {
  __shared__ uint8_t t[HT + 2][HT + 2];
  const int b = blockIdx.z;
  const int y0 = blockIdx.y * HT, x0 = blockIdx.x * HT;
  uint8_t* img = lab + (int64_t)b * H * W;
  for (int e = threadIdx.x; e < (HT + 2) * (HT + 2); e += blockDim.x) {
    const int ty = e / (HT + 2), tx = e - ty * (HT + 2);
    const int y = y0 + ty - 1, x = x0 + tx - 1;
    t[ty][tx] = (y >= 0 && y < H && x >= 0 && x < W) ? img[(int64_t)y * W + x] : 0;
  }
  __syncthreads();
  bool any = false;
  for (;;) {
    bool local = false;
    for (int e = threadIdx.x; e < HT * HT; e += blockDim.x) {
      const int ty = e / HT + 1, tx = e % HT + 1;
      if (t[ty][tx] != 1) continue;
      bool s = false;
#pragma unroll
      for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
        for (int dx = -1; dx <= 1; ++dx) s |= t[ty + dy][tx + dx] == 2;
      if (s) {
        t[ty][tx] = 2;
        local = true;
      }
    }
    if (!__syncthreads_or(local)) break;
    any = true;
  }
  if (any) {
    for (int e = threadIdx.x; e < HT * HT; e += blockDim.x) {
      const int ty = e / HT, tx = e % HT;
      const int y = y0 + ty, x = x0 + tx;
      if (y < H && x < W && t[ty + 1][tx + 1] == 2 && img[(int64_t)y * W + x] != 2) {
        img[(int64_t)y * W + x] = 2;
        *changed = 1;
      }
    }
  }
}

// Quad-tree per max cell: thread = min cell; counts of edge pixels (label 2), pyramid in
// shared memory, then every min cell walks down from the max cell (split iff side > min
// and count > thr * area, in double) and flags the leaf at its top-left min cell.
__global__ void quadtree_kernel(const uint8_t* __restrict__ lab, int H, int W, int mn, int levels, double thr,
                                int hr, int wr, const int32_t* __restrict__ ext, int32_t* __restrict__ flag) {
  // hr x wr (or ext[2 b], ext[2 b + 1] per image): the min cells of the real field (the rest is
  // edge padding): leaves whose top-left cell lies in the padding are not emitted
  extern __shared__ int cnt[];           // pyramid: level l has (R >> l)^2 entries
  const int R = 1 << (levels - 1);       // min cells per max-cell side
  const int b = blockIdx.z;
  if (ext) {
    hr = ext[2 * b];
    wr = ext[2 * b + 1];
  }
  const int cy0 = blockIdx.y * R, cx0 = blockIdx.x * R;   // first min cell of the max cell
  const int Wc = W / mn, Hc = H / mn;
  const uint8_t* img = lab + (int64_t)b * H * W;
  int* lvl[8];
  {
    int off = 0;
    for (int l = 0; l < levels; ++l) {
      lvl[l] = cnt + off;
      off += (R >> l) * (R >> l);
    }
  }
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int cy = e / R, cx = e % R;
    int c = 0;
    for (int yy = 0; yy < mn; ++yy)
      for (int xx = 0; xx < mn; ++xx)
        c += img[(int64_t)((cy0 + cy) * mn + yy) * W + (cx0 + cx) * mn + xx] == 2;
    lvl[0][e] = c;
  }
  __syncthreads();
  for (int l = 1; l < levels; ++l) {
    const int n = R >> l;
    for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
      const int y = e / n, x = e % n, m2 = 2 * n;
      const int* p = lvl[l - 1];
      lvl[l][e] = p[(2 * y) * m2 + 2 * x] + p[(2 * y) * m2 + 2 * x + 1] + p[(2 * y + 1) * m2 + 2 * x] +
                  p[(2 * y + 1) * m2 + 2 * x + 1];
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < R * R; e += blockDim.x) {
    const int cy = e / R, cx = e % R;
    int l = levels - 1;
    for (; l > 0; --l) {
      const int n = R >> l, side = mn << l;
      const int c = lvl[l][(cy >> l) * n + (cx >> l)];
      if (!((double)c > thr * (double)side * (double)side)) break;
    }
    const bool origin = ((cy & ((1 << l) - 1)) == 0) && ((cx & ((1 << l) - 1)) == 0) && cy0 + cy < hr &&
                        cx0 + cx < wr;
    flag[((int64_t)b * Hc + cy0 + cy) * Wc + cx0 + cx] = origin ? (mn << l) : 0;
  }
}

// exclusive scan of (flag != 0) over n entries in three passes (block sums of 1024)
constexpr int SCAN_B = 1024;
__global__ void scan_blocks_kernel(const int32_t* __restrict__ flag, int64_t n, int32_t* __restrict__ bsum) {
  const int64_t i = (int64_t)blockIdx.x * SCAN_B + threadIdx.x;
  const int v = __syncthreads_count((i < n && flag[i] != 0) ? 1 : 0);
  if (threadIdx.x == 0) bsum[blockIdx.x] = v;
}

__global__ void edges_kernel(const uint8_t* __restrict__ lab, uint8_t* __restrict__ e, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    e[i] = lab[i] == 2 ? 1 : 0;
}
__global__ void scan_sums_kernel(int32_t* __restrict__ bsum, int64_t nb, int32_t* __restrict__ total) {
  // one block: exclusive scan of nb block sums, in chunks of 1024
  __shared__ int s[SCAN_B];
  int carry = 0;
  for (int64_t base = 0; base < nb; base += SCAN_B) {
    const int64_t i = base + threadIdx.x;
    const int v = i < nb ? bsum[i] : 0;
    s[threadIdx.x] = v;
    __syncthreads();
    for (int off = 1; off < SCAN_B; off <<= 1) {
      const int add = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
      __syncthreads();
      s[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < nb) bsum[i] = carry + s[threadIdx.x] - v;
    const int tot = s[SCAN_B - 1];
    __syncthreads();
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}
__global__ void scatter_kernel(const int32_t* __restrict__ flag, int64_t n, const int32_t* __restrict__ bsum,
                               int Hc, int Wc, int mn, int32_t* __restrict__ patches, int32_t* __restrict__ offsets) {
  __shared__ int s[SCAN_B];
  const int64_t i = (int64_t)blockIdx.x * SCAN_B + threadIdx.x;
  const int f = i < n ? flag[i] : 0;
  const int v = f != 0 ? 1 : 0;
  s[threadIdx.x] = v;
  __syncthreads();
  for (int off = 1; off < SCAN_B; off <<= 1) {
    const int add = threadIdx.x >= off ? s[threadIdx.x - off] : 0;
    __syncthreads();
    s[threadIdx.x] += add;
    __syncthreads();
  }
  const int pos = bsum[blockIdx.x] + s[threadIdx.x] - v;
  if (i < n) {
    const int64_t per = (int64_t)Hc * Wc;
    const int b = (int)(i / per);
    const int64_t rem = i - (int64_t)b * per;
    const int cy = (int)(rem / Wc), cx = (int)(rem - (int64_t)cy * Wc);
    if (rem == 0) offsets[b] = pos;             // first leaf of image b (its cell (0,0) is always an origin)
    if (v) {
      int32_t* p = patches + (int64_t)pos * 4;
      p[0] = b;
      p[1] = cy * mn;
      p[2] = cx * mn;
      p[3] = f;
    }
  }
}

// tokens as one GEMM: the pooled leaf row [C m m | one-hot(level)] times [W_tok | E_scale^T]
// (the scale embedding rides on the one-hot columns), + b_tok.  One warp per leaf here.
__global__ void pool_kernel(const float* __restrict__ feat, const int32_t* __restrict__ patches, int n, int C, int H,
                            int W, int m, int levels, float* __restrict__ rows, int ldr) {
  const int leaf = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (leaf >= n) return;
  const int32_t* p = patches + (int64_t)leaf * 4;
  const int b = p[0], r = p[1], c = p[2], s = p[3];
  const int f = s / m, K = C * m * m;
  const float inv = 1.f / (float)(f * f);
  float* row = rows + (int64_t)leaf * ldr;
  for (int e = lane; e < K; e += 32) {
    const int ch = e / (m * m), ij = e - ch * m * m, i = ij / m, j = ij - i * m;
    const float* src = feat + (((int64_t)b * C + ch) * H + r + i * f) * W + c + j * f;
    float acc = 0.f;
    for (int yy = 0; yy < f; ++yy)
      for (int xx = 0; xx < f; ++xx) acc += __ldg(src + (int64_t)yy * W + xx);
    row[e] = acc * inv;
  }
  int lvl = 0;
  while ((m << lvl) < s) ++lvl;
  for (int e = lane; e < levels; e += 32) row[K + e] = e == lvl ? 1.f : 0.f;
}

// W_ext [D][K + levels] = [W_tok | E_scale^T]
__global__ void wext_kernel(const float* __restrict__ wt, const float* __restrict__ es, int D, int K, int levels,
                            float* __restrict__ wext) {
  const int ld = K + levels;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < (int64_t)D * ld;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(e / ld), k = (int)(e - (int64_t)o * ld);
    wext[e] = k < K ? wt[(int64_t)o * K + k] : es[(int64_t)(k - K) * D + o];
  }
}

// decompression: proj rows [n][C m m] (one GEMM) broadcast nearest over each leaf
__global__ void broadcast_kernel(const float* __restrict__ proj, const int32_t* __restrict__ patches, int C, int H,
                                 int W, int m, float* __restrict__ img) {
  const int32_t* p = patches + (int64_t)blockIdx.x * 4;
  const int b = p[0], r = p[1], c = p[2], s = p[3];
  const float* pr = proj + (int64_t)blockIdx.x * C * m * m;
  const int64_t px = (int64_t)C * s * s;
  for (int64_t e = threadIdx.x; e < px; e += blockDim.x) {
    const int ch = (int)(e / ((int64_t)s * s));
    const int rem = (int)(e - (int64_t)ch * s * s);
    const int y = rem / s, x = rem - y * s;
    img[(((int64_t)b * C + ch) * H + r + y) * W + c + x] = __ldg(pr + (ch * m + (y * m) / s) * m + (x * m) / s);
  }
}

// out = b + sum W[o][i][dy][dx] in[i][y+dy-1][x+dx-1] (zero padding), per image
__global__ void smooth_kernel(const float* __restrict__ in, const float* __restrict__ ws, const float* __restrict__ bs,
                              float* __restrict__ out, int C, int H, int W) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y;
  const int bo = blockIdx.z, b = bo / C, o = bo - b * C;
  if (x >= W) return;
  float acc = __ldg(bs + o);
  for (int i = 0; i < C; ++i) {
    const float* src = in + ((int64_t)b * C + i) * H * W;
    const float* w = ws + ((int64_t)o * C + i) * 9;
#pragma unroll
    for (int dy = 0; dy < 3; ++dy) {
      const int yy = y + dy - 1;
      if (yy < 0 || yy >= H) continue;
#pragma unroll
      for (int dx = 0; dx < 3; ++dx) {
        const int xx = x + dx - 1;
        if (xx < 0 || xx >= W) continue;
        acc = fmaf(__ldg(w + dy * 3 + dx), __ldg(src + (int64_t)yy * W + xx), acc);
      }
    }
  }
  out[(((int64_t)b * C + o) * H + y) * W + x] = acc;
}

}  // namespace

// ---- R41 / R42: compression inside the Reslim forward, per (sample, tile) image ----
// image i = b T + t: the tile's padded rectangle (pad_h x pad_w patches) of sample b; its
// z0 rows are b chunk_tokens + (tok_off - tok0) + u pad_w + w (the forward's packing)
__device__ __forceinline__ int64_t z0_row(const ChunkDev& ch, const DevTile& t, int b, int u, int w) {
  return (int64_t)b * ch.chunk_tokens + (t.tok_off - ch.tok0) + (int64_t)u * t.pad_w + w;
}

// f[i][y][x] = mean_d z0[row(i, min(y, pad_h - 1), min(x, pad_w - 1))][d]  (edge padding to Hq x Wq)
__global__ void cfield_kernel(const float* __restrict__ z0, ChunkDev ch, int T, int B, int D, int Hq, int Wq,
                              float* __restrict__ f) {
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= (int64_t)B * T * Hq * Wq) return;
  const int img = (int)(warp / ((int64_t)Hq * Wq));
  const int rem = (int)(warp - (int64_t)img * Hq * Wq);
  const int b = img / T, ti = img - b * T;
  const DevTile t = ch.tiles[ch.tb + ti];
  const int u = min(rem / Wq, t.pad_h - 1), w = min(rem % Wq, t.pad_w - 1);
  const float* row = z0 + z0_row(ch, t, b, u, w) * D;
  float s = 0.f;
  for (int d = lane; d < D; d += 32) s += row[d];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) f[warp] = s / D;
}

// token of a leaf = mean of z0 over its patches inside the rectangle + E_scale[log2 side]
__global__ void ctoken_kernel(const float* __restrict__ z0, ChunkDev ch, int T, const int32_t* __restrict__ leaves,
                              int D, const float* __restrict__ es, float* __restrict__ tok) {
  const int32_t* p = leaves + (int64_t)blockIdx.x * 4;
  const int img = p[0], u0 = p[1], w0 = p[2], s = p[3];
  const int b = img / T;
  const DevTile t = ch.tiles[ch.tb + img - b * T];
  const int u1 = min(u0 + s, t.pad_h), w1 = min(w0 + s, t.pad_w);
  const float inv = 1.f / (float)((u1 - u0) * (w1 - w0));
  int lvl = 0;
  while ((1 << lvl) < s) ++lvl;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    float acc = 0.f;
    for (int u = u0; u < u1; ++u)
      for (int w = w0; w < w1; ++w) acc += __ldg(z0 + z0_row(ch, t, b, u, w) * D + d);
    tok[(int64_t)blockIdx.x * D + d] = acc * inv + __ldg(es + (int64_t)lvl * D + d);
  }
}

// decompression: every CORE patch of a leaf gets the leaf's head output row, at its row of
// tile_out [B][chunk core tokens][Nh] (the halo patches are discarded)
__global__ void decompress_kernel(const __nv_bfloat16* __restrict__ g, ChunkDev ch, int T,
                                  const int32_t* __restrict__ leaves, int Nh, __nv_bfloat16* __restrict__ tile_out) {
  const int32_t* p = leaves + (int64_t)blockIdx.x * 4;
  const int img = p[0], s = p[3];
  const int b = img / T;
  const DevTile t = ch.tiles[ch.tb + img - b * T];
  const int cy = t.core_y0 - t.pad_y0, cx = t.core_x0 - t.pad_x0;   // core rect in rectangle coordinates
  const int u0 = max(p[1], cy), w0 = max(p[2], cx);
  const int u1 = min(p[1] + s, cy + t.core_h), w1 = min(p[2] + s, cx + t.core_w);
  if (u1 <= u0 || w1 <= w0) return;
  const int nw = w1 - w0, npatch = (u1 - u0) * nw;
  const int64_t base = (int64_t)b * ch.chunk_core + (t.core_off - ch.core0);
  if (Nh % 8 == 0) {                                 // 16-byte rows: vector copies
    const int n8 = Nh / 8;
    const uint4* src = reinterpret_cast<const uint4*>(g + (int64_t)blockIdx.x * Nh);
    for (int e = threadIdx.x; e < npatch * n8; e += blockDim.x) {
      const int q = e / n8, c = e - q * n8;
      const int u = u0 + q / nw, w = w0 + q % nw;
      reinterpret_cast<uint4*>(tile_out + (base + (int64_t)(u - cy) * t.core_w + (w - cx)) * Nh)[c] = __ldg(src + c);
    }
  } else {
    const __nv_bfloat16* src = g + (int64_t)blockIdx.x * Nh;
    for (int e = threadIdx.x; e < npatch * Nh; e += blockDim.x) {
      const int q = e / Nh, c = e - q * Nh;
      const int u = u0 + q / nw, w = w0 + q % nw;
      tile_out[(base + (int64_t)(u - cy) * t.core_w + (w - cx)) * Nh + c] = src[c];
    }
  }
}

bool compress_taps(float sigma, float* w, int* r) {
  const int rr = (int)std::ceil(3.0 * sigma);
  if (!(sigma > 0.f) || 2 * rr + 1 > MAX_TAPS) return false;
  double s = 0.0, t[MAX_TAPS];
  for (int i = -rr; i <= rr; ++i) s += (t[i + rr] = std::exp(-(double)(i * i) / (2.0 * sigma * sigma)));
  for (int i = 0; i < 2 * rr + 1; ++i) w[i] = (float)(t[i] / s);
  *r = rr;
  return true;
}

void launch_canny(const float* img, float* tmp, float* tmp2, float* mag, uint8_t* dir, uint8_t* lab, unsigned* gmax,
                  int* changed, int B, int H, int W, float sigma, float low_frac, float high_frac, cudaStream_t st,
                  int* passes) {
  Taps t{};
  compress_taps(sigma, t.w, &t.r);
  const dim3 blk(128), grid((W + 127) / 128, H, B);
  blur_h_kernel<<<grid, blk, 0, st>>>(img, tmp, H, W, t);
  blur_v_kernel<<<grid, blk, 0, st>>>(tmp, tmp2, H, W, t);
  cudaMemsetAsync(gmax, 0, sizeof(unsigned) * B, st);
  sobel_kernel<<<grid, blk, 0, st>>>(tmp2, mag, dir, H, W, gmax);
  nms_kernel<<<grid, blk, 0, st>>>(mag, dir, lab, H, W, gmax, low_frac, high_frac);
  const dim3 hg((W + HT - 1) / HT, (H + HT - 1) / HT, B);
  int n = 0;
  for (;;) {
    int h_changed = 0;
    cudaMemsetAsync(changed, 0, sizeof(int), st);
    hyst_kernel<<<hg, HT * 8, 0, st>>>(lab, H, W, changed);
    cudaMemcpyAsync(&h_changed, changed, sizeof(int), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    ++n;
    if (!h_changed || n > H * W) break;
  }
  if (passes) *passes = n;
}

void launch_quadtree(const uint8_t* lab, int32_t* flag, int32_t* bsum, int32_t* total, int32_t* patches,
                     int32_t* offsets, int B, int H, int W, int mn, int mx, double thr, cudaStream_t st, int hr,
                     int wr, const int32_t* ext) {
  if (hr <= 0) hr = H / mn;
  if (wr <= 0) wr = W / mn;
  int levels = 1;
  while ((mn << (levels - 1)) < mx) ++levels;
  const int R = 1 << (levels - 1);
  int words = 0;
  for (int l = 0; l < levels; ++l) words += (R >> l) * (R >> l);
  const dim3 grid(W / mx, H / mx, B);
  quadtree_kernel<<<grid, std::min(R * R, 1024), words * sizeof(int), st>>>(lab, H, W, mn, levels, thr, hr, wr,
                                                                            ext, flag);
  const int64_t n = (int64_t)B * (H / mn) * (W / mn);
  const int64_t nb = (n + SCAN_B - 1) / SCAN_B;
  scan_blocks_kernel<<<(unsigned)nb, SCAN_B, 0, st>>>(flag, n, bsum);
  scan_sums_kernel<<<1, SCAN_B, 0, st>>>(bsum, nb, total);
  scatter_kernel<<<(unsigned)nb, SCAN_B, 0, st>>>(flag, n, bsum, H / mn, W / mn, mn, patches, offsets);
}

void launch_edges(const uint8_t* lab, uint8_t* e, int64_t n, cudaStream_t st) {
  edges_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(lab, e, n);
}

void launch_tokenize(const float* feat, const int32_t* patches, int n, int C, int H, int W, int m, int D,
                     int levels, const float* wt, const float* bt, const float* es, float* rows, float* wext,
                     float* tok, cudaStream_t st) {
  const int K = C * m * m, ld = K + levels;
  wext_kernel<<<(unsigned)std::min<int64_t>(((int64_t)D * ld + 255) / 256, 1024), 256, 0, st>>>(wt, es, D, K, levels,
                                                                                            wext);
  if (n <= 0) return;
  pool_kernel<<<(n + 7) / 8, 256, 0, st>>>(feat, patches, n, C, H, W, m, levels, rows, ld);
  EpiParams ep{};
  ep.M = n; ep.N = D; ep.bias = bt; ep.C = tok; ep.ldc = D;
  launch_sgemm(EPI_BIAS, rows, ld, wext, ld, n, D, ld, ep, st);
}

void launch_detokenize(const float* tok, const int32_t* patches, int n, int B, int C, int H, int W, int m, int D,
                       const float* wd, const float* bd, const float* ws, const float* bs, float* proj, float* work,
                       float* out, cudaStream_t st) {
  if (n > 0) {
    const int K = C * m * m;
    EpiParams ep{};
    ep.M = n; ep.N = K; ep.bias = bd; ep.C = proj; ep.ldc = K;
    launch_sgemm(EPI_BIAS, tok, D, wd, D, n, K, D, ep, st);
    broadcast_kernel<<<n, 256, 0, st>>>(proj, patches, C, H, W, m, work);
  }
  smooth_kernel<<<dim3((W + 127) / 128, H, B * C), 128, 0, st>>>(work, ws, bs, out, C, H, W);
}

void launch_cfield(const float* z0, const ChunkDev& ch, int T, int B, int D, int Hq, int Wq, float* f,
                   cudaStream_t st) {
  const int64_t warps = (int64_t)B * T * Hq * Wq;
  cfield_kernel<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(z0, ch, T, B, D, Hq, Wq, f);
}

void launch_ctokens(const float* z0, const ChunkDev& ch, int T, const int32_t* leaves, int n, int D, const float* es,
                    float* tok, cudaStream_t st) {
  if (n > 0) ctoken_kernel<<<n, std::min(D, 256), 0, st>>>(z0, ch, T, leaves, D, es, tok);
}

void launch_decompress(const __nv_bfloat16* g, const ChunkDev& ch, int T, const int32_t* leaves, int n, int Nh,
                       __nv_bfloat16* tile_out, cudaStream_t st) {
  if (n > 0) decompress_kernel<<<n, 128, 0, st>>>(g, ch, T, leaves, Nh, tile_out);
}

}  // namespace orbit2
