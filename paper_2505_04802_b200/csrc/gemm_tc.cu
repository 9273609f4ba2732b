// gemm_tc.cu -- bf16 GEMM on 5th-generation tensor cores (tcgen05) for the
// dense contractions of the Reslim forward (patch embed, QKV, O-projection,
// MLP up/down, decoder head):
//     C[M,N] = A[M,K] . W[N,K]^T    (W = PyTorch Linear weight [out][in])
// with the epilogue fused: bias, exact-erf GELU (R9), fp32 residual add, or
// the embedding epilogue (bias + resolution embedding + sincos position, R7/R8).
//
// Structure (persistent, one CTA per SM, warp-specialised):
//   warp 0 lane 0 : TMA producer, STAGES-deep smem ring (SWIZZLE_128B, BK = 64)
//   warp 1 lane 0 : tcgen05.mma issuer (M=128, N=BN, K=16 per instruction),
//                   accumulator in TMEM, double-buffered (2 x BN fp32 columns)
//   warp 2        : TMEM allocator
//   warps 4-11    : epilogue (2 warpgroups, one per column half), tcgen05.ld
//                   32x32b -> registers -> fused op -> global
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <mutex>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

// ---------------------------------------------------------------------------
// TMA descriptor encoding through the driver entry point (no -lcuda)
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
static std::once_flag g_encode_once;

static void load_encode() {
  cudaDriverEntryPointQueryResult q;
  void* fn = nullptr;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
      q == cudaDriverEntryPointSuccess)
    g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

bool tma_available() {
  std::call_once(g_encode_once, load_encode);
  return g_encode != nullptr;
}

// 2-D bf16 row-major tensor [rows][ld] (cols used = cols), box [box_rows][box_cols]
bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz) {
  if (!tma_available()) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS && std::getenv("ORBIT2_DEBUG_TMAP"))
    std::fprintf(stderr, "[orbit2] cuTensorMapEncodeTiled(bf16) = %d: ptr %p dims %lld x %lld ld %lld box %d x %d swz %d\n",
                 (int)r, ptr, (long long)cols, (long long)rows, (long long)ld, box_cols, box_rows, (int)swz);
  return r == CUDA_SUCCESS;
}

// 2-D fp32 row-major tensor [rows][ld], box [box_rows][box_cols]
bool make_tmap_f32(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                   int box_cols, CUtensorMapSwizzle swz) {
  if (!tma_available()) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 4)};
  cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

// ---------------------------------------------------------------------------
// Per-device launch state (a process may drive several devices: attributes and
// SM counts are per device, cached by device ordinal)
// ---------------------------------------------------------------------------
// 3-D fp32 tensor [d2][d1][d0] (d0 contiguous), box [b2][b1][b0], no swizzle:
// the smem box is dense [b2][b1][b0]; out-of-bound elements are zero-filled.
bool make_tmap_f32_3d(CUtensorMap* map, const void* ptr, int64_t d0, int64_t d1, int64_t d2, int b0, int b1,
                      int b2) {
  if (!tma_available()) return false;
  cuuint64_t dims[3] = {(cuuint64_t)d0, (cuuint64_t)d1, (cuuint64_t)d2};
  cuuint64_t strides[2] = {(cuuint64_t)(d0 * 4), (cuuint64_t)(d0 * d1 * 4)};
  cuuint32_t box[3] = {(cuuint32_t)b0, (cuuint32_t)b1, (cuuint32_t)b2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

namespace {
constexpr int kMaxDev = 64;
std::atomic<int> g_sms[kMaxDev];
std::mutex g_attr_mu;
}  // namespace

int num_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return 148;
  int n = g_sms[dev].load(std::memory_order_relaxed);
  if (n <= 0) {
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    g_sms[dev].store(n, std::memory_order_relaxed);
  }
  return n;
}

bool smem_attr_once(const void* func, int bytes, std::atomic<uint64_t>* done) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return false;
  const uint64_t bit = 1ull << dev;
  if (done->load(std::memory_order_acquire) & bit) return true;
  std::lock_guard<std::mutex> lk(g_attr_mu);
  if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes) != cudaSuccess) return false;
  done->fetch_or(bit, std::memory_order_release);
  return true;
}

namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int LN_CHUNK_BYTES = BM * 32 * 4;   // *_LN staging: 128 rows x 32 fp32 columns (16 KB)
// *_LN staging buffers per warpgroup: the embedding epilogue (K = Din: a short main loop, the
// epilogue is the kernel) keeps 4 so a chunk's store rarely waits for the one before last to
// have read its buffer; the residual form keeps 2 (its z loads are tied to 2 barriers)
#ifndef ORBIT2_EMBED_LN_BUFS
#define ORBIT2_EMBED_LN_BUFS 4
#endif
template <int EPI>
__host__ __device__ constexpr int ln_bufs() { return EPI == EPI_EMBED_LN ? ORBIT2_EMBED_LN_BUFS : 2; }

template <int EPI, bool OUT_BF16>
__device__ __forceinline__ void epilogue_chunk(const EpiParams& ep, int64_t row, int n0, const uint32_t (&r)[32]) {
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  const bool full = n0 + 32 <= ep.N;
  if constexpr (EPI == EPI_DGELU) {
  } else if (full) {
    const float4* b4 = reinterpret_cast<const float4*>(ep.bias + n0);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 bb = __ldg(b4 + j);
      v[4 * j] += bb.x; v[4 * j + 1] += bb.y; v[4 * j + 2] += bb.z; v[4 * j + 3] += bb.w;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (n0 + j < ep.N) v[j] += __ldg(ep.bias + n0 + j);
  }
  if constexpr (EPI == EPI_GELU) {
    if (ep.aux) {   // training: keep GELU'(pre-activation) for the backward
      __nv_bfloat16* h = reinterpret_cast<__nv_bfloat16*>(const_cast<void*>(ep.aux)) + row * ep.ldc + n0;
      for (int j = 0; j < 32; ++j)
        if (n0 + j < ep.N) {
          const float x = v[j];
          h[j] = __float2bfloat16_rn(0.5f * (1.0f + erff(x * 0.70710678118654752f)) +
                                     x * 0.39894228040143268f * __expf(-0.5f * x * x));
        }
    }
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = 0.5f * v[j] * (1.0f + erff(v[j] * 0.70710678118654752f));
  }
  if constexpr (EPI == EPI_DGELU) {   // v = acc (no bias): dh = dgelu * GELU'(h) (aux = GELU'(h))
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(ep.aux) + row * ep.ldc + n0;
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] *= n0 + j < ep.N ? __bfloat162float(h[j]) : 0.f;
  }
  if constexpr (EPI == EPI_BIAS || EPI == EPI_GELU || EPI == EPI_DGELU) {
    if constexpr (OUT_BF16) {
      __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(ep.C) + row * ep.ldc + n0;
      if (full) {
        uint4* c4 = reinterpret_cast<uint4*>(c);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 w;
          w.x = tc::pack_bf16(v[8 * j + 0], v[8 * j + 1]);
          w.y = tc::pack_bf16(v[8 * j + 2], v[8 * j + 3]);
          w.z = tc::pack_bf16(v[8 * j + 4], v[8 * j + 5]);
          w.w = tc::pack_bf16(v[8 * j + 6], v[8 * j + 7]);
          c4[j] = w;
        }
      } else {
        for (int j = 0; j < 32; ++j)
          if (n0 + j < ep.N) c[j] = __float2bfloat16_rn(v[j]);
      }
    } else {
      float* c = reinterpret_cast<float*>(ep.C) + row * ep.ldc + n0;
      if (full) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          reinterpret_cast<float4*>(c)[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
      } else {
        for (int j = 0; j < 32; ++j)
          if (n0 + j < ep.N) c[j] = v[j];
      }
    }
  } else if constexpr (EPI == EPI_RESID) {
    float* z = reinterpret_cast<float*>(ep.C) + row * ep.ldc + n0;
    const float* zs = ep.aux ? reinterpret_cast<const float*>(ep.aux) + row * ep.ldc + n0 : z;
    if (full) {
      float4* z4 = reinterpret_cast<float4*>(z);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        float4 o = reinterpret_cast<const float4*>(zs)[j];
        o.x += v[4 * j]; o.y += v[4 * j + 1]; o.z += v[4 * j + 2]; o.w += v[4 * j + 3];
        z4[j] = o;
      }
    } else {
      for (int j = 0; j < 32; ++j)
        if (n0 + j < ep.N) z[j] = zs[j] + v[j];
    }
  } else {  // EPI_EMBED: z = acc + bias + pi(u,w); 32-column chunks never straddle D/2 (D % 64 == 0)
    const int2 uw = __ldg(ep.rowinfo + row);
    const float* pe = n0 < ep.half ? ep.pos_u + (int64_t)(uw.x + ep.pos_off) * ep.half + n0
                                   : ep.pos_w + (int64_t)(uw.y + ep.pos_off) * ep.half + (n0 - ep.half);
    float* z = reinterpret_cast<float*>(ep.C) + row * ep.ldc + n0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float4 p4 = __ldg(reinterpret_cast<const float4*>(pe) + j);
      reinterpret_cast<float4*>(z)[j] =
          make_float4(v[4 * j] + p4.x, v[4 * j + 1] + p4.y, v[4 * j + 2] + p4.z, v[4 * j + 3] + p4.w);
    }
  }
}

#ifndef ORBIT2_GEMM_WS
#define ORBIT2_GEMM_WS 1
#endif
#ifndef ORBIT2_GEMM_PAIR   // 0: single-CTA tiles only (A/B builds)
#define ORBIT2_GEMM_PAIR 1
#endif
// Epilogue global loads one chunk ahead (A/B, profiles/r02bl): the GELU' chunk of the DGELU
// epilogue gains (C2 training dx_mlp_down 10.38 -> 10.04 ms); the residual z chunk of the
// transposed residual GEMMs loses (C3 O-projection 6.90 -> 7.25 ms), so it is off.
#ifndef ORBIT2_EPI_PREFETCH_A
#define ORBIT2_EPI_PREFETCH_A 1
#endif
#ifndef ORBIT2_EPI_PREFETCH_Z
#define ORBIT2_EPI_PREFETCH_Z 0
#endif
#ifndef ORBIT2_PAIR_STAGES   // ring depth of the pair tiles (the residual GEMMs take one more)
#define ORBIT2_PAIR_STAGES 4
#endif
#ifndef ORBIT2_GEMM_GELU_TANH   // tanh-form GELU (reading R28) in the inference MLP-up epilogue
#define ORBIT2_GEMM_GELU_TANH 1
#endif

template <int BN, int STAGES, int EPI, bool OUT_BF16, bool TRANS, bool WS = false, bool PAIR = false>
__global__ void __launch_bounds__(384, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmD, int64_t M,
                   int64_t Ncols, int K, EpiParams ep) {
  // Persistent: CTA c owns output tiles c, c + gridDim.x, ...  Normal mode:
  // m-major, n fastest (consecutive CTAs share the activation block through
  // L2).  TRANS mode computes C^T = W X^T (A = weight rows, B = tokens) so the
  // epilogue's fp32 residual update is coalesced; tiles are token-major.
  // bf16 outputs leave through shared memory and TMA stores (full lines).  The TMA ring
  // runs continuously across tiles; the fp32 accumulator is double-buffered
  // in TMEM (2 x BN columns) so the epilogue of tile i overlaps the MMAs of
  // tile i+1.
  // WS (weight-stationary, K == 256): the CTA's BN x K weight slice is loaded once
  // into shared memory and every tile of the CTA (the grid is a multiple of the
  // number of column tiles, so a CTA keeps one column tile) streams only its
  // activation block through the ring: 3x less L2 -> SM traffic for the QKV GEMM.
  constexpr int A_BYTES = BM * BK * 2;
  // PAIR (cta_group::2 on a 2-CTA cluster): a tile is 2 BM kernel rows x BN; CTA r loads A rows
  // [m0 + BM r, + BM) and B rows [n0 + BN/2 r, + BN/2), the leader issues M = 2 BM MMAs, and
  // each CTA's TMEM / epilogue holds its own BM rows: 2/3 of the L2 -> SM operand bytes per FLOP.
  constexpr int BNL = PAIR ? BN / 2 : BN;   // B rows this CTA loads
  constexpr int PM = PAIR ? 2 * BM : BM;    // kernel rows per tile
  constexpr int B_BYTES = BNL * BK * 2;
  static_assert(!PAIR || (!WS && EPI != EPI_RESID_LN && EPI != EPI_EMBED_LN), "pair: plain epilogues only");
  constexpr int WS_K = 256;
  constexpr int B_RING = WS ? (WS_K / BK) : STAGES;   // B atoms resident (WS) or ring slots
  constexpr uint32_t TMEM_COLS = 2 * BN;
  constexpr bool LN = EPI == EPI_RESID_LN || EPI == EPI_EMBED_LN;
  // GELU: a second staging set for the training forward's GELU' store (aux)
  constexpr int LNB = ln_bufs<EPI>();
  constexpr int STG_BYTES = LN ? 2 * LNB * LN_CHUNK_BYTES : (EPI == EPI_GELU ? 2 : 1) * 8 * 2 * 2048;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align inside the __shared__ array (keeps the shared address space: STS, not generic ST)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + B_RING * B_BYTES + STG_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;    // [2] accumulator ready
  uint64_t* tempty = tfull + 2;        // [2] accumulator drained
  uint64_t* zfull = tempty + 2;        // *_LN: [2 warpgroups][2] z chunk landed
  uint64_t* wfull = zfull + 4;         // WS: weight slice landed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(wfull + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr bool TMA_OUT = (EPI == EPI_BIAS || EPI == EPI_GELU || EPI == EPI_DGELU) && OUT_BF16 && !TRANS;
  const int nk = K / BK;
  const int64_t num_n = (Ncols + BN - 1) / BN;
  const int64_t num_m = (M + PM - 1) / PM;
  const int64_t num_tiles = num_m * num_n;
  auto tile_mn = [&](int64_t tile, int64_t& m0, int64_t& n0) {
    if (TRANS) { m0 = (tile % num_m) * PM; n0 = (tile / num_m) * BN; }
    else       { m0 = (tile / num_n) * PM; n0 = (tile % num_n) * BN; }
  };
  const uint32_t rank = PAIR ? tc::cluster_ctarank() : 0u;
  const int64_t t_first = PAIR ? (int64_t)(blockIdx.x >> 1) : (int64_t)blockIdx.x;   // pair index
  const int64_t t_step = PAIR ? (int64_t)(gridDim.x >> 1) : (int64_t)gridDim.x;
  uint8_t* stg = sB + B_RING * B_BYTES;   // TMA-store staging: 8 warps x 2 x (32 x 32 bf16);
                                          // *_LN: 2 warpgroups x 2 x (128 x 32 fp32)

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmA);
    tc::prefetch_tmap(&tmB);
    if (TMA_OUT || LN) tc::prefetch_tmap(&tmC);
    if (EPI == EPI_GELU || LN) tc::prefetch_tmap(&tmD);
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&tfull[s], 1);
      // *_LN: one warpgroup drains a buffer; PAIR: one arrive per epilogue warp of both CTAs
      tc::mbar_init(&tempty[s], PAIR ? 16 : LN ? 128 : 256);
    }
    for (int s = 0; s < 4; ++s) tc::mbar_init(&zfull[s], 1);
    tc::mbar_init(wfull, 1);
    tc::fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (PAIR) tc::tmem_alloc_pair(tmem_slot, TMEM_COLS);
    else tc::tmem_alloc(tmem_slot, TMEM_COLS);
  }
  tc::tc_fence_before();
  if constexpr (PAIR) tc::cluster_sync();   // both CTAs' barriers initialised before any remote signal
  else __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      uint32_t it = 0;
      if (WS && blockIdx.x < num_tiles) {   // the CTA's weight slice, once
        int64_t m0, n0;
        tile_mn(blockIdx.x, m0, n0);
        tc::mbar_arrive_expect_tx(wfull, B_RING * B_BYTES);
        for (int kb = 0; kb < B_RING; ++kb) tc::tma_load_2d(&tmB, sB + kb * B_BYTES, wfull, kb * BK, (int32_t)n0);
      }
      for (int64_t tile = t_first; tile < num_tiles; tile += t_step) {
        int64_t m0, n0;
        tile_mn(tile, m0, n0);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
          tc::mbar_wait(&empty[s], ph ^ 1);
          if constexpr (PAIR) {   // both halves complete on the leader's full barrier
            if (rank == 0) tc::mbar_arrive_expect_tx(&full[s], 2 * (A_BYTES + B_BYTES));
            const uint32_t fb = tc::map_rank(tc::smem_u32(&full[s]), 0);
            tc::tma_load_2d_pair(&tmA, sA + s * A_BYTES, fb, kb * BK, (int32_t)(m0 + rank * BM));
            tc::tma_load_2d_pair(&tmB, sB + s * B_BYTES, fb, kb * BK, (int32_t)(n0 + rank * BNL));
            continue;
          }
          tc::mbar_arrive_expect_tx(&full[s], WS ? A_BYTES : A_BYTES + B_BYTES);
          tc::tma_load_2d(&tmA, sA + s * A_BYTES, &full[s], kb * BK, (int32_t)m0);
          if (!WS) tc::tma_load_2d(&tmB, sB + s * B_BYTES, &full[s], kb * BK, (int32_t)n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      // ---------------- MMA issuer (PAIR: the leader CTA only) ----------------
      constexpr uint32_t idesc = tc::idesc_bf16(PM, BN, 0, 0);
      uint32_t it = 0, lt = 0;
      if (WS) tc::mbar_wait(wfull, 0);
      for (int64_t tile = t_first; tile < num_tiles; tile += t_step, ++lt) {
        const uint32_t buf = lt & 1;
        tc::mbar_wait(&tempty[buf], ((lt >> 1) & 1) ^ 1);
        tc::tc_fence_after();
        const uint32_t acc = tmem + buf * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const uint32_t s = it % STAGES, ph = (it / STAGES) & 1;
          tc::mbar_wait(&full[s], ph);
          tc::tc_fence_after();
          const uint32_t a0 = tc::smem_u32(sA + s * A_BYTES), b0 = tc::smem_u32(sB + (WS ? kb : s) * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            const uint64_t ad = tc::sdesc(a0 + kk * 32, 16, 1024, tc::SW_128B);
            const uint64_t bd = tc::sdesc(b0 + kk * 32, 16, 1024, tc::SW_128B);
            if constexpr (PAIR) tc::mma_bf16_ss_pair(acc, ad, bd, idesc, (kb | kk) != 0);
            else tc::mma_bf16_ss(acc, ad, bd, idesc, (kb | kk) != 0);
          }
          if constexpr (PAIR) tc::mma_commit_pair(&empty[s]);   // frees the stage in both CTAs
          else tc::mma_commit(&empty[s]);
        }
        if constexpr (PAIR) tc::mma_commit_pair(&tfull[buf]);
        else tc::mma_commit(&tfull[buf]);
      }
    }
  } else if (LN && warp >= 4) {
    // ---------------- LayerNorm-fused epilogue (BN == N == 256) ----------------
    // Warpgroup wg owns TMEM buffer wg, i.e. every other tile; thread = row
    // (TMEM lane), so the row statistics are thread-local.  Pass 1 over 8 chunks
    // of 32 columns: z_new = acc + bias + (z | pi), written back to TMEM and
    // stored through swizzled smem + TMA (z chunks of the RESID form arrive by
    // TMA two chunks ahead); pass 2: sum (z_new - mean)^2 from TMEM (two-pass
    // variance, as the LN kernel); pass 3: LN -> bf16 -> smem -> TMA store xn.
    const int wg = (warp - 4) >> 2;
    const int q = warp & 3;
    const int rr = q * 32 + lane;                       // row within the tile
    const bool issuer = q == 0 && lane == 0;
    const uint32_t nb = 1 + wg;                         // named barrier of this warpgroup
    uint8_t* zb = stg + wg * LNB * LN_CHUNK_BYTES;
    uint64_t* zf = zfull + wg * 2;
    uint32_t zuse[2] = {0, 0};                          // loads completed per buffer (parity)
    uint32_t lt = 0;
    for (int64_t tile = t_first; tile < num_tiles; tile += t_step, ++lt) {
      if ((int)(lt & 1) != wg) continue;
      const uint32_t buf = lt & 1;
      int64_t m0, n0;
      tile_mn(tile, m0, n0);
      const int64_t row = m0 + rr;
      auto load_z = [&](int c) {                        // issuer only
        tc::bulk_wait_read<0>();                        // the buffer's previous store has read it
        tc::mbar_arrive_expect_tx(&zf[c & 1], LN_CHUNK_BYTES);
        tc::tma_load_2d(&tmC, zb + (c & 1) * LN_CHUNK_BYTES, &zf[c & 1], c * 32, (int32_t)m0);
      };
      if (EPI == EPI_RESID_LN && issuer) {
        load_z(0);
        load_z(1);
      }
      tc::mbar_wait(&tfull[buf], (lt >> 1) & 1);
      tc::tc_fence_after();
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + buf * BN;
      int2 uw = make_int2(0, 0);
      if (EPI == EPI_EMBED_LN && row < M) uw = __ldg(ep.rowinfo + row);
      float sum = 0.f;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint8_t* sb = zb + (c % LNB) * LN_CHUNK_BYTES + rr * 128;   // this row's 128 bytes (SW128)
        if (EPI == EPI_RESID_LN) {
          tc::mbar_wait(&zf[c & 1], zuse[c & 1] & 1);
          ++zuse[c & 1];
        } else {                                         // staging reuse: the buffer's last store has read it
          if (issuer) tc::bulk_wait_read<LNB - 1>();
          asm volatile("bar.sync %0, 128;" ::"r"(nb) : "memory");
        }
        uint32_t r[32];
        tc::tmem_ld32(taddr + c * 32, r);
        tc::tmem_ld_wait();
        float v[32];
        const float4* b4 = reinterpret_cast<const float4*>(ep.bias + c * 32);
        const float* pe = nullptr;
        if (EPI == EPI_EMBED_LN)
          pe = c * 32 < ep.half ? ep.pos_u + (int64_t)(uw.x + ep.pos_off) * ep.half + c * 32
                                : ep.pos_w + (int64_t)(uw.y + ep.pos_off) * ep.half + (c * 32 - ep.half);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const float4 bb = __ldg(b4 + u);
          float4 a;
          if (EPI == EPI_RESID_LN) a = *reinterpret_cast<const float4*>(sb + ((u ^ (rr & 7)) << 4));
          else a = __ldg(reinterpret_cast<const float4*>(pe) + u);
          v[4 * u] = __uint_as_float(r[4 * u]) + bb.x + a.x;
          v[4 * u + 1] = __uint_as_float(r[4 * u + 1]) + bb.y + a.y;
          v[4 * u + 2] = __uint_as_float(r[4 * u + 2]) + bb.z + a.z;
          v[4 * u + 3] = __uint_as_float(r[4 * u + 3]) + bb.w + a.w;
          *reinterpret_cast<float4*>(sb + ((u ^ (rr & 7)) << 4)) =
              make_float4(v[4 * u], v[4 * u + 1], v[4 * u + 2], v[4 * u + 3]);
        }
        float s4[4] = {0.f, 0.f, 0.f, 0.f};    // 4 partial sums: no 256-long chain of dependent adds
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          s4[j & 3] += v[j];
          r[j] = __float_as_uint(v[j]);
        }
        sum += (s4[0] + s4[1]) + (s4[2] + s4[3]);
        tc::tmem_st32(taddr + c * 32, r);
        tc::fence_proxy_async_smem();
        asm volatile("bar.sync %0, 128;" ::"r"(nb) : "memory");
        if (issuer) {
          tc::tma_store_2d(&tmC, zb + (c % LNB) * LN_CHUNK_BYTES, c * 32, (int32_t)m0);
          tc::bulk_commit();
          if (EPI == EPI_RESID_LN && c + 2 < 8) load_z(c + 2);
        }
      }
      tc::tmem_st_wait();
      const float mean = sum * (1.0f / 256.0f);
      float var = 0.f;
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t r[32];
        tc::tmem_ld32(taddr + c * 32, r);
        tc::tmem_ld_wait();
        float v4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float d = __uint_as_float(r[j]) - mean;
          v4[j & 3] = fmaf(d, d, v4[j & 3]);
        }
        var += (v4[0] + v4[1]) + (v4[2] + v4[3]);
      }
      const float rstd = rsqrtf(var * (1.0f / 256.0f) + 1e-5f);
#pragma unroll 1
      for (int c = 0; c < 8; ++c) {
        uint32_t r[32];
        tc::tmem_ld32(taddr + c * 32, r);
        tc::tmem_ld_wait();
        if (c == 7) {                                   // accumulator buffer drained
          tc::tc_fence_before();
          tc::mbar_arrive(&tempty[buf]);
        }
        uint8_t* sb = zb + (c % LNB) * LN_CHUNK_BYTES;    // bf16 box [128 rows][64 B], SWIZZLE_64B
        if (issuer) tc::bulk_wait_read<LNB - 1>();
        asm volatile("bar.sync %0, 128;" ::"r"(nb) : "memory");
        const float4* g4 = reinterpret_cast<const float4*>(ep.ln_g + c * 32);
        const float4* e4 = reinterpret_cast<const float4*>(ep.ln_b + c * 32);
        uint8_t* srow = sb + rr * 64;
        const int sw = (rr >> 1) & 3;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint32_t w[4];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const float4 gg = __ldg(g4 + 2 * u + h), ee = __ldg(e4 + 2 * u + h);
            const int j = 8 * u + 4 * h;
            w[2 * h] = tc::pack_bf16((__uint_as_float(r[j]) - mean) * rstd * gg.x + ee.x,
                                     (__uint_as_float(r[j + 1]) - mean) * rstd * gg.y + ee.y);
            w[2 * h + 1] = tc::pack_bf16((__uint_as_float(r[j + 2]) - mean) * rstd * gg.z + ee.z,
                                         (__uint_as_float(r[j + 3]) - mean) * rstd * gg.w + ee.w);
          }
          *reinterpret_cast<uint4*>(srow + ((u ^ sw) << 4)) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        tc::fence_proxy_async_smem();
        asm volatile("bar.sync %0, 128;" ::"r"(nb) : "memory");
        if (issuer) {
          tc::tma_store_2d(&tmD, sb, c * 32, (int32_t)m0);
          tc::bulk_commit();
        }
      }
    }
    if (issuer) tc::bulk_wait_all();
  } else if (warp >= 4) {
    // ---------------- epilogue: 2 warpgroups, each half of the columns ----------------
    const int q = warp & 3;                  // TMEM lane quarter of this warp
    const int half = (warp - 4) >> 2;        // column half
    uint8_t* my_stg = stg + (warp - 4) * 2 * 2048;
    uint32_t lt = 0, nst = 0;
    for (int64_t tile = t_first; tile < num_tiles; tile += t_step, ++lt) {
      const uint32_t buf = lt & 1;
      int64_t m0, n0;
      tile_mn(tile, m0, n0);
      m0 += rank * BM;                       // PAIR: this CTA's rows of the tile
      tc::mbar_wait(&tfull[buf], (lt >> 1) & 1);
      tc::tc_fence_after();
      const int64_t row = m0 + q * 32 + lane;
      const uint32_t taddr = tmem + ((uint32_t)(q * 32) << 16) + buf * BN;
      // Loads the epilogue needs from global memory (TRANS: the residual z chunk; DGELU: the
      // GELU' chunk) are issued one chunk ahead, so their latency overlaps the current chunk.
      constexpr bool PF_Z = ORBIT2_EPI_PREFETCH_Z && TRANS && EPI == EPI_RESID;
      constexpr bool PF_A = ORBIT2_EPI_PREFETCH_A && TMA_OUT && EPI == EPI_DGELU;
      float zpf[PF_Z ? 32 : 1];
      uint4 apf[PF_A ? 4 : 1];
      auto z_full = [&](int c) { return row < M && n0 + c + 32 <= ep.M; };
      auto z_src = [&](int c) {
        return ep.aux ? reinterpret_cast<const float*>(ep.aux) + (n0 + c) * ep.ldc + row
                      : reinterpret_cast<const float*>(ep.C) + (n0 + c) * ep.ldc + row;
      };
      auto a_full = [&](int c) { return row < M && n0 + c + 32 <= ep.N; };
      auto prefetch = [&](int c) {
        if constexpr (PF_Z) {
          if (z_full(c)) {
            const float* zs = z_src(c);
#pragma unroll
            for (int j = 0; j < 32; ++j) zpf[j] = zs[(int64_t)j * ep.ldc];
          }
        }
        if constexpr (PF_A) {
          if (a_full(c)) {
            const uint4* a4 = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(ep.aux) +
                                                             row * ep.ldc + n0 + c);
#pragma unroll
            for (int u = 0; u < 4; ++u) apf[u] = __ldg(a4 + u);
          }
        }
      };
      prefetch(half * (BN / 2));
#pragma unroll 1
      for (int c0 = half * (BN / 2); c0 < (half + 1) * (BN / 2); c0 += 32) {
        float zcur[PF_Z ? 32 : 1];
        uint4 acur[PF_A ? 4 : 1];
        if constexpr (PF_Z) {
#pragma unroll
          for (int j = 0; j < 32; ++j) zcur[j] = zpf[j];
        }
        if constexpr (PF_A) {
#pragma unroll
          for (int u = 0; u < 4; ++u) acur[u] = apf[u];
        }
        if (c0 + 32 < (half + 1) * (BN / 2)) prefetch(c0 + 32);
        uint32_t r[32];
        tc::tmem_ld32(taddr + c0, r);
        tc::tmem_ld_wait();
        if (c0 + 32 >= (half + 1) * (BN / 2)) {   // my half read: hand the buffer back
          tc::tc_fence_before();
          if constexpr (PAIR) {                   // to the leader's barrier, one arrive per warp
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_cluster(tc::map_rank(tc::smem_u32(&tempty[buf]), 0));
          } else {
            tc::mbar_arrive(&tempty[buf]);
          }
        }
        if constexpr (TRANS) {
          // rows = output features, columns = tokens: z[t][f] += acc + bias[f]
          if (row < M) {
            const float bf = __ldg(ep.bias + row);
            float* zc = reinterpret_cast<float*>(ep.C) + (n0 + c0) * ep.ldc + row;
            // training: residual input from aux (the forward keeps z_in), else in place
            const float* zs = ep.aux ? reinterpret_cast<const float*>(ep.aux) + (n0 + c0) * ep.ldc + row : zc;
            const int64_t t0 = n0 + c0;
            if (t0 + 32 <= ep.M) {
              float zv[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) zv[j] = PF_Z ? zcur[PF_Z ? j : 0] : zs[(int64_t)j * ep.ldc];
#pragma unroll
              for (int j = 0; j < 32; ++j) zc[(int64_t)j * ep.ldc] = zv[j] + (__uint_as_float(r[j]) + bf);
            } else {
              for (int j = 0; j < 32; ++j)
                if (t0 + j < ep.M) zc[(int64_t)j * ep.ldc] = zs[(int64_t)j * ep.ldc] + (__uint_as_float(r[j]) + bf);
            }
          }
        } else if constexpr (TMA_OUT) {
          if (n0 + c0 < ep.N) {
            float v[32];
            if constexpr (EPI == EPI_DGELU) {   // dh = acc * GELU'(h): aux row chunk (64 B)
              float gd[32];
              if (row < M && n0 + c0 + 32 <= ep.N) {
                const uint4* a4 = reinterpret_cast<const uint4*>(reinterpret_cast<const __nv_bfloat16*>(ep.aux) +
                                                                 row * ep.ldc + n0 + c0);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                  const uint4 w = PF_A ? acur[PF_A ? u : 0] : __ldg(a4 + u);
                  const __nv_bfloat162* hp = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
                  for (int e = 0; e < 4; ++e) {
                    const float2 f = __bfloat1622float2(hp[e]);
                    gd[8 * u + 2 * e] = f.x;
                    gd[8 * u + 2 * e + 1] = f.y;
                  }
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  gd[j] = (row < M && n0 + c0 + j < ep.N)
                              ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(ep.aux)[row * ep.ldc + n0 + c0 + j])
                              : 0.f;
              }
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]) * gd[j];
            } else if (n0 + c0 + 32 <= ep.N) {
              const float4* b4 = reinterpret_cast<const float4*>(ep.bias + n0 + c0);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 bb = __ldg(b4 + j);
                v[4 * j] = __uint_as_float(r[4 * j]) + bb.x;
                v[4 * j + 1] = __uint_as_float(r[4 * j + 1]) + bb.y;
                v[4 * j + 2] = __uint_as_float(r[4 * j + 2]) + bb.z;
                v[4 * j + 3] = __uint_as_float(r[4 * j + 3]) + bb.w;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                v[j] = __uint_as_float(r[j]) + (n0 + c0 + j < ep.N ? __ldg(ep.bias + n0 + c0 + j) : 0.f);
            }
            const bool keep_grad = EPI == EPI_GELU && ep.aux != nullptr;   // training forward
            float gd[EPI == EPI_GELU ? 32 : 1];
            if constexpr (EPI == EPI_GELU) {
              if (keep_grad) {
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                  float2 g2, d2;
                  tc::gelu2_and_grad_fast(make_float2(v[j], v[j + 1]), g2, d2);
                  v[j] = g2.x; v[j + 1] = g2.y; gd[j] = d2.x; gd[j + 1] = d2.y;
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; j += 2) {   // packed f32x2: half the FMA-pipe issues
                  const float2 g2 = ORBIT2_GEMM_GELU_TANH ? tc::gelu2_tanh_fast(make_float2(v[j], v[j + 1]))
                                                          : tc::gelu2_erf_fast(make_float2(v[j], v[j + 1]));
                  v[j] = g2.x; v[j + 1] = g2.y;
                }
              }
            }
            uint8_t* sb = my_stg + (nst & 1) * 2048;
            if (lane == 0) tc::bulk_wait_read<1>();   // this buffer's previous store has read it
            __syncwarp();
            uint8_t* srow = sb + lane * 64;
            const int sw = (lane >> 1) & 3;           // SWIZZLE_64B pattern of the TMA box
#pragma unroll
            for (int u = 0; u < 4; ++u)
              *reinterpret_cast<uint4*>(srow + ((u ^ sw) << 4)) =
                  make_uint4(tc::pack_bf16(v[8 * u], v[8 * u + 1]), tc::pack_bf16(v[8 * u + 2], v[8 * u + 3]),
                             tc::pack_bf16(v[8 * u + 4], v[8 * u + 5]), tc::pack_bf16(v[8 * u + 6], v[8 * u + 7]));
            if constexpr (EPI == EPI_GELU) {
              if (keep_grad) {   // GELU'(pre-activation) -> aux through the second staging set
                uint8_t* grow = sb + 8 * 2 * 2048 + lane * 64;
#pragma unroll
                for (int u = 0; u < 4; ++u)
                  *reinterpret_cast<uint4*>(grow + ((u ^ sw) << 4)) =
                      make_uint4(tc::pack_bf16(gd[8 * u], gd[8 * u + 1]), tc::pack_bf16(gd[8 * u + 2], gd[8 * u + 3]),
                                 tc::pack_bf16(gd[8 * u + 4], gd[8 * u + 5]),
                                 tc::pack_bf16(gd[8 * u + 6], gd[8 * u + 7]));
              }
            }
            tc::fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tc::tma_store_2d(&tmC, sb, (int32_t)(n0 + c0), (int32_t)(m0 + q * 32));
              if (keep_grad) tc::tma_store_2d(&tmD, sb + 8 * 2 * 2048, (int32_t)(n0 + c0), (int32_t)(m0 + q * 32));
              tc::bulk_commit();
            }
            ++nst;
          }
        } else {
          if (row < M && n0 + c0 < ep.N) epilogue_chunk<EPI, OUT_BF16>(ep, row, (int)(n0 + c0), r);
        }
      }
    }
    if (TMA_OUT && lane == 0) tc::bulk_wait_all();
  }
  tc::tc_fence_before();
  if constexpr (PAIR) tc::cluster_sync();   // neither CTA leaves while the pair's MMAs / arrives target it
  else __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    if constexpr (PAIR) tc::tmem_dealloc_pair(tmem, TMEM_COLS);
    else tc::tmem_dealloc(tmem, TMEM_COLS);
  }
}

template <int BN, int STAGES, int EPI, bool OUT_BF16, bool TRANS = false, bool WS = false, bool PAIR = false>
bool launch_impl(const GemmOperand& A, const GemmOperand& Bw, int64_t M, int64_t N, int64_t K, const EpiParams& ep,
                 cudaStream_t st) {
  // normal: kernel rows = activations A (M), cols = weights Bw (N)
  // TRANS : kernel rows = weights Bw (N features), cols = activations A (M tokens)
  const GemmOperand& ka = TRANS ? Bw : A;
  const GemmOperand& kb = TRANS ? A : Bw;
  const int64_t Mk = TRANS ? N : M, Nk = TRANS ? M : N;
  CUtensorMap ta, tb, tcm, tdm;
  // an operand may hold fewer than K valid columns (the patch matrix: Din of
  // round_up(Din, 64)); the TMA zero-fills the rest of the K range
  if (!make_tmap_bf16(&ta, ka.ptr, ka.rows, ka.cols ? ka.cols : K, ka.ld, BM, BK, CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  constexpr int BNL = PAIR ? BN / 2 : BN;
  if (!make_tmap_bf16(&tb, kb.ptr, kb.rows, kb.cols ? kb.cols : K, kb.ld, BNL, BK, CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  constexpr bool TMA_OUT = (EPI == EPI_BIAS || EPI == EPI_GELU || EPI == EPI_DGELU) && OUT_BF16 && !TRANS;
  constexpr bool LN = EPI == EPI_RESID_LN || EPI == EPI_EMBED_LN;
  tcm = ta;   // unused unless set below
  tdm = ta;
  if (TMA_OUT) {
    if (!make_tmap_bf16(&tcm, ep.C, M, N, ep.ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B)) return false;
    if (EPI == EPI_GELU && ep.aux != nullptr &&   // training forward: GELU' store
        !make_tmap_bf16(&tdm, ep.aux, M, N, ep.ldc, 32, 32, CU_TENSOR_MAP_SWIZZLE_64B))
      return false;
  }
  if (LN) {   // z fp32 [M][N] in 128 x 32 boxes (SW128), xn bf16 [M][N] in 128 x 32 boxes (SW64)
    if (!make_tmap_f32(&tcm, ep.C, M, N, ep.ldc, BM, 32, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
    if (!make_tmap_bf16(&tdm, ep.xn, M, N, N, BM, 32, CU_TENSOR_MAP_SWIZZLE_64B)) return false;
  }
  constexpr int STG = LN ? 2 * ln_bufs<EPI>() * LN_CHUNK_BYTES : (EPI == EPI_GELU ? 2 : 1) * 8 * 2 * 2048;
  constexpr int smem = STAGES * BM * BK * 2 + (WS ? 256 / BK : STAGES) * BNL * BK * 2 + STG + 1024 + 256;
  static_assert(smem <= 227 * 1024, "shared memory");
  if (WS && K != 256) return false;
  auto kern = gemm_tc_kernel<BN, STAGES, EPI, OUT_BF16, TRANS, WS, PAIR>;
  static std::atomic<uint64_t> attr_done{0};   // per instantiation, per device
  if (!smem_attr_once(reinterpret_cast<const void*>(kern), smem, &attr_done)) return false;
  const int64_t num_n = (Nk + BN - 1) / BN;
  if (PAIR) {   // 2-CTA clusters, one pair per tile in flight: grid = 2 x min(tiles, SMs / 2)
    const int64_t tiles = ((Mk + 2 * BM - 1) / (2 * BM)) * num_n;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(2 * std::min<int64_t>(tiles, num_sms() / 2)));
    cfg.blockDim = dim3(384);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, ta, tb, tcm, tdm, Mk, Nk, (int)K, ep) == cudaSuccess;
  }
  const int64_t tiles = ((Mk + BM - 1) / BM) * num_n;
  int grid = (int)std::min<int64_t>(tiles, num_sms());
  if (WS) grid = (int)std::max<int64_t>(num_n, grid / num_n * num_n);   // a CTA keeps one column tile
  kern<<<grid, 384, smem, st>>>(ta, tb, tcm, tdm, Mk, Nk, (int)K, ep);
  return true;
}

}  // namespace

bool launch_gemm_tc(int epi, int out_bf16, const GemmOperand& A, const GemmOperand& Bw, int64_t M, int64_t N,
                    int64_t K, const EpiParams& ep, cudaStream_t st) {
  if (K % BK != 0 || M <= 0 || N <= 0) return false;
  if (epi == EPI_RESID_LN || epi == EPI_EMBED_LN) {   // whole rows in one 256-column tile
    if (N != 256 || ep.ldc != 256) return false;
    return epi == EPI_RESID_LN ? launch_impl<256, 3, EPI_RESID_LN, false>(A, Bw, M, N, K, ep, st)
                               : launch_impl<256, (ORBIT2_EMBED_LN_BUFS > 2 ? 2 : 3), EPI_EMBED_LN, false>(A, Bw, M, N, K, ep, st);
  }
  // CTA pairs (cta_group::2) for BN = 256 GEMMs with at least one 256 x 256 tile per pair:
  // the large GEMMs at D >= 1024 are bound by the L2 -> SM operand stream (~15.4 TB/s,
  // profiles/r02az), which a pair cuts to 2/3 per FLOP
  // (K >= 512: with 4 K-steps per tile the pair's longer tiles lose more than the operand
  // savings win -- the D = 256 training GEMMs with K = 256 measured 6-10 % slower, r02bc)
  auto pair_ok = [&](int64_t Mk, int64_t Nk) {
    return ORBIT2_GEMM_PAIR && !ep.single_cta && K >= 512 && ((Mk + 255) / 256) * ((Nk + 255) / 256) >= num_sms() / 2;
  };
  // Residual update: transposed tiles (features on TMEM lanes) for coalesced z.
  if (epi == EPI_RESID && N % BM == 0) {
    if (pair_ok(N, M)) return launch_impl<256, ORBIT2_PAIR_STAGES + 1, EPI_RESID, false, true, false, true>(A, Bw, M, N, K, ep, st);
    return launch_impl<256, 3, EPI_RESID, false, true>(A, Bw, M, N, K, ep, st);
  }
  // BN = 256 halves the shared-memory operand traffic per FLOP; 128 when N is
  // not a multiple of 256 (e.g. the decoder head, K*P*P = 192).
  if (N % 256 == 0) {
    constexpr int BN = 256, ST = 3;
    if (pair_ok(M, N) && !(epi == EPI_BIAS && out_bf16 && K == 256 && ORBIT2_GEMM_WS)) {
      switch (epi) {
        case EPI_BIAS:
          return out_bf16 ? launch_impl<BN, ORBIT2_PAIR_STAGES, EPI_BIAS, true, false, false, true>(A, Bw, M, N, K, ep, st)
                          : launch_impl<BN, ORBIT2_PAIR_STAGES, EPI_BIAS, false, false, false, true>(A, Bw, M, N, K, ep, st);
        case EPI_GELU: return launch_impl<BN, ORBIT2_PAIR_STAGES, EPI_GELU, true, false, false, true>(A, Bw, M, N, K, ep, st);
        case EPI_RESID: return launch_impl<BN, ORBIT2_PAIR_STAGES + 1, EPI_RESID, false, false, false, true>(A, Bw, M, N, K, ep, st);
        case EPI_EMBED: return launch_impl<BN, ORBIT2_PAIR_STAGES, EPI_EMBED, false, false, false, true>(A, Bw, M, N, K, ep, st);
        case EPI_DGELU: return launch_impl<BN, ORBIT2_PAIR_STAGES, EPI_DGELU, true, false, false, true>(A, Bw, M, N, K, ep, st);
      }
    }
    switch (epi) {
      case EPI_BIAS:
        if (out_bf16 && K == 256 && ORBIT2_GEMM_WS)   // QKV at D = 256: weight-stationary
          return launch_impl<BN, 4, EPI_BIAS, true, false, true>(A, Bw, M, N, K, ep, st);
        return out_bf16 ? launch_impl<BN, ST, EPI_BIAS, true>(A, Bw, M, N, K, ep, st)
                        : launch_impl<BN, ST, EPI_BIAS, false>(A, Bw, M, N, K, ep, st);
      case EPI_GELU: return launch_impl<BN, ST, EPI_GELU, true>(A, Bw, M, N, K, ep, st);
      case EPI_RESID: return launch_impl<BN, ST, EPI_RESID, false>(A, Bw, M, N, K, ep, st);
      case EPI_EMBED: return launch_impl<BN, ST, EPI_EMBED, false>(A, Bw, M, N, K, ep, st);
      case EPI_DGELU: return launch_impl<BN, ST, EPI_DGELU, true>(A, Bw, M, N, K, ep, st);
    }
  } else {
    constexpr int BN = 128, ST = 5;
    switch (epi) {
      case EPI_BIAS:
        return out_bf16 ? launch_impl<BN, ST, EPI_BIAS, true>(A, Bw, M, N, K, ep, st)
                        : launch_impl<BN, ST, EPI_BIAS, false>(A, Bw, M, N, K, ep, st);
      case EPI_GELU: return launch_impl<BN, ST, EPI_GELU, true>(A, Bw, M, N, K, ep, st);
      case EPI_RESID: return launch_impl<BN, ST, EPI_RESID, false>(A, Bw, M, N, K, ep, st);
      case EPI_EMBED: return launch_impl<BN, ST, EPI_EMBED, false>(A, Bw, M, N, K, ep, st);
    }
  }
  return false;
}

}  // namespace orbit2
