// mlp_tc.cu -- fused transformer MLP on tcgen05 for D = 256 (the 9.5M-class
// Reslim):   z += W_2 . GELU(W_1 . x + b_1) + b_2      (R9, exact-erf GELU)
// with x = LN2(z) in bf16.  The 128 x 1024 hidden tile of a row block never
// leaves the SM: S_h = X W_1[h]^T lands in TMEM, 8 epilogue warps apply
// bias + GELU and write bf16 H_h into shared memory (SW128 K-major), and the
// tensor core accumulates O += H_h W_2[:,h]^T in TMEM.  Saves the 2 x 4D x 2 B
// per token hidden-activation round trip through HBM of the unfused pair.
//
// Persistent, one CTA per SM, warp-specialised (128 + 128 EW threads):
//   warp 0 lane 0 : TMA producer: X tile (64 KB) per row block, then W_1 / W_2
//                   slices (32 KB slots) through a 3-slot ring, in the order the
//                   MMA consumes them: W1(0) W1(1) W2(0) W1(2) W2(1) ... W2(7)
//   warp 1 lane 0 : MMA issuer: GEMM1(h) into S buffer h&1 (2 x 128 TMEM cols),
//                   GEMM2(h-1) transposed: O^T = W_2 H^T into 2 x 128 TMEM cols
//                   (features on TMEM lanes, tokens on columns: coalesced z update)
//   warp 2        : TMEM allocator (512 columns)
//   warps 4..     : epilogue, EW warpgroups (HC / EW hidden columns each): bias +
//                   GELU in packed f32x2 arithmetic; at the end of a row block
//                   O^T + b_2 is staged in the (then idle) H buffers and added to
//                   z by bulk reduce-add copies (the L2 does the read-modify-write
//                   while the warps start the next block)
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

long long* g_mlp_timeline = nullptr;   // debug: set by orbit2_debug_mlp_timeline

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz);

namespace {

constexpr int BM = 128;
constexpr int DM = 256;         // model width D
constexpr int FH = 1024;        // hidden width 4D
constexpr int HC = 128;         // hidden chunk
constexpr int NCH = FH / HC;    // 8 chunks
constexpr int RS = 3;           // ring slots
constexpr int SLOT = 32768;
constexpr int X_BYTES = BM * DM * 2;     // 64 KB
constexpr int H_BYTES = BM * HC * 2;     // 32 KB
constexpr int SMEM = X_BYTES + 2 * H_BYTES + RS * SLOT + 1024 + 512;
#ifndef ORBIT2_MLP_EPI_WG
#define ORBIT2_MLP_EPI_WG 2   // 4 measured no faster (the GELU is FMA-pipe bound, not latency bound)
#endif
constexpr int EW = ORBIT2_MLP_EPI_WG;   // epilogue warpgroups (4 warps each: the TMEM lane quarters)
constexpr int CW = HC / EW;              // hidden columns per warpgroup and chunk
constexpr int ET = 128 * EW;             // epilogue threads
constexpr int THREADS = 128 + ET;

// debug timeline (-DORBIT2_MLP_TIMELINE): tl[(role * 64 + chunk) * 8 + event], CTA 0
#ifdef ORBIT2_MLP_TIMELINE
#define MTL(role, c, ev)                                                                              \
  do {                                                                                                \
    if (tl != nullptr && blockIdx.x == 0 && (c) < 64) tl[((role) * 64 + (c)) * 8 + (ev)] = clock64(); \
  } while (0)
#else
#define MTL(role, c, ev) \
  do {                   \
  } while (0)
#endif

__global__ void __launch_bounds__(THREADS, 1)
    mlp_tc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                  const __grid_constant__ CUtensorMap tmW2, const float* __restrict__ b1,
                  const float* __restrict__ b2, float* __restrict__ z, int64_t M, long long* __restrict__ tl) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align inside the __shared__ array (keeps the shared address space: STS, not generic ST)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;
  uint8_t* sH = sX + X_BYTES;          // [2][H_BYTES]
  uint8_t* sW = sH + 2 * H_BYTES;      // [RS][SLOT]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sW + RS * SLOT);
  uint64_t* x_full = bar;
  uint64_t* x_free = x_full + 1;
  uint64_t* w_full = x_free + 1;       // [RS]
  uint64_t* w_empty = w_full + RS;     // [RS]
  uint64_t* s_full = w_empty + RS;     // [2]
  uint64_t* s_free = s_full + 2;       // [2]
  uint64_t* h_full = s_free + 2;       // [2]
  uint64_t* h_free = h_full + 2;       // [2]
  uint64_t* o_full = h_free + 2;
  uint64_t* o_free = o_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t num_tiles = (M + BM - 1) / BM;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmX);
    tc::prefetch_tmap(&tmW1);
    tc::prefetch_tmap(&tmW2);
    tc::mbar_init(x_full, 1);
    tc::mbar_init(x_free, 1);
    for (int s = 0; s < RS; ++s) {
      tc::mbar_init(&w_full[s], 1);
      tc::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&s_full[s], 1);
      tc::mbar_init(&s_free[s], ET);
      tc::mbar_init(&h_full[s], ET);
      tc::mbar_init(&h_free[s], 1);
    }
    tc::mbar_init(o_full, 1);
    tc::mbar_init(o_free, ET);
    tc::fence_barrier_init();
  }
  if (warp == 2) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      uint32_t it = 0, tl_ = 0;
      auto slot_begin = [&]() -> uint8_t* {
        const uint32_t s = it % RS, ph = (it / RS) & 1;
        tc::mbar_wait(&w_empty[s], ph ^ 1);
        tc::mbar_arrive_expect_tx(&w_full[s], SLOT);
        return sW + s * SLOT;
      };
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl_) {
        const int32_t m0 = (int32_t)(tile * BM);
        tc::mbar_wait(x_free, (tl_ & 1) ^ 1);
        tc::mbar_arrive_expect_tx(x_full, X_BYTES);
        for (int a = 0; a < DM / 64; ++a) tc::tma_load_2d(&tmX, sX + a * 16384, x_full, a * 64, m0);
        for (int s = 0; s <= NCH; ++s) {
          if (s < NCH) {
            for (int pr = 0; pr < 2; ++pr, ++it) {   // W1 rows s*128.., K slices 2pr, 2pr+1
              uint8_t* dst = slot_begin();
              uint64_t* fb = &w_full[it % RS];
              tc::tma_load_2d(&tmW1, dst, fb, (2 * pr) * 64, s * HC);
              tc::tma_load_2d(&tmW1, dst + 16384, fb, (2 * pr + 1) * 64, s * HC);
            }
          }
          if (s >= 1) {
            const int h = s - 1;
            for (int k2 = 0; k2 < 2; ++k2, ++it) {    // W2 all 256 rows, K slice h*128 + 64*k2
              uint8_t* dst = slot_begin();
              uint64_t* fb = &w_full[it % RS];
              tc::tma_load_2d(&tmW2, dst, fb, h * HC + k2 * 64, 0);
              tc::tma_load_2d(&tmW2, dst + 16384, fb, h * HC + k2 * 64, 128);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer ----------------
      constexpr uint32_t id1 = tc::idesc_bf16(BM, HC, 0, 0);
      constexpr uint32_t id2 = tc::idesc_bf16(128, BM, 0, 0);   // O^T half: 128 features x 128 tokens
      const uint32_t x_addr = tc::smem_u32(sX), h_addr = tc::smem_u32(sH), w_addr = tc::smem_u32(sW);
      uint32_t it = 0, tl_ = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl_) {
        tc::mbar_wait(x_full, tl_ & 1);
        tc::tc_fence_after();
        for (int s = 0; s <= NCH; ++s) {
          if (s < NCH) {
            const uint32_t gc = tl_ * NCH + s, buf = gc & 1, use = gc >> 1;
            MTL(0, gc, 0);
            if (use >= 1) tc::mbar_wait(&s_free[buf], (use - 1) & 1);
            MTL(0, gc, 1);
            tc::tc_fence_after();
            for (int pr = 0; pr < 2; ++pr, ++it) {
              const uint32_t sl = it % RS;
              tc::mbar_wait(&w_full[sl], (it / RS) & 1);
              tc::tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {     // two 64-wide K slices per slot
                const int ks = 2 * pr + (kk >> 2);
                const uint64_t ad = tc::sdesc(x_addr + ks * 16384 + (kk & 3) * 32, 16, 1024, tc::SW_128B);
                const uint64_t bd =
                    tc::sdesc(w_addr + sl * SLOT + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024, tc::SW_128B);
                tc::mma_bf16_ss(tmem + buf * HC, ad, bd, id1, (pr | kk) != 0);
              }
              tc::mma_commit(&w_empty[sl]);
            }
            tc::mma_commit(&s_full[buf]);
            MTL(0, gc, 2);
            if (s == NCH - 1) tc::mma_commit(x_free);
          }
          if (s >= 1) {
            const int h = s - 1;
            const uint32_t gc = tl_ * NCH + h, hb = gc & 1;
            tc::mbar_wait(&h_full[hb], (gc >> 1) & 1);
            if (h == 0) tc::mbar_wait(o_free, (tl_ & 1) ^ 1);
            MTL(0, gc, 3);
            tc::tc_fence_after();
            for (int k2 = 0; k2 < 2; ++k2, ++it) {
              const uint32_t sl = it % RS;
              tc::mbar_wait(&w_full[sl], (it / RS) & 1);
              tc::tc_fence_after();
#pragma unroll
              for (int kk = 0; kk < 8; ++kk) {     // O^T[f,t] += W2[f, hidden] H[t, hidden]
                const int half = kk >> 2;
                const uint64_t ad =
                    tc::sdesc(w_addr + sl * SLOT + half * 16384 + (kk & 3) * 32, 16, 1024, tc::SW_128B);
                const uint64_t bd =
                    tc::sdesc(h_addr + hb * H_BYTES + k2 * 16384 + (kk & 3) * 32, 16, 1024, tc::SW_128B);
                tc::mma_bf16_ss(tmem + 256 + half * 128, ad, bd, id2, (h | k2 | (kk & 3)) != 0);
              }
              tc::mma_commit(&w_empty[sl]);
            }
            tc::mma_commit(&h_free[hb]);
            MTL(0, gc, 4);
            if (h == NCH - 1) tc::mma_commit(o_full);
          }
        }
      }
    }
  } else if (warp >= 4) {
    // ---------------- epilogue: EW warpgroups ----------------
    const int q = warp & 3;
    const int wg = (warp - 4) >> 2;
    const int r = q * 32 + lane;                 // row within the block = TMEM lane
    const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
    const bool issuer = warp == 4 && lane == 0;   // issues the residual bulk reductions
    uint32_t tl_ = 0;
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl_) {
      for (int h = 0; h < NCH; ++h) {
        const uint32_t gc = tl_ * NCH + h, buf = gc & 1, use = gc >> 1;
        const bool st = warp == 4 && lane == 0;
        if (st) MTL(1, gc, 0);
        tc::mbar_wait(&s_full[buf], use & 1);
        if (st) MTL(1, gc, 1);
        tc::tc_fence_after();
        float v[CW];
#pragma unroll
        for (int c = 0; c < CW; c += 32)
          tc::tmem_ld32(lane_addr + buf * HC + wg * CW + c, *reinterpret_cast<uint32_t(*)[32]>(v + c));
        tc::tmem_ld_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&s_free[buf]);
        if (use >= 1) tc::mbar_wait(&h_free[buf], (use - 1) & 1);
        if (st) MTL(1, gc, 2);
        const float4* bb = reinterpret_cast<const float4*>(b1 + h * HC + wg * CW);
        // SW128 K-major H: 64-column atoms of 16 KB, 16-byte units XOR-swizzled by row
        uint8_t* hrow = sH + buf * H_BYTES + ((wg * CW) >> 6) * 16384 + r * 128;
        const int u0 = ((wg * CW) & 63) >> 3;
        uint32_t hv[CW / 2];   // bf16 GELU outputs, packed pairs
#pragma unroll
        for (int c8 = 0; c8 < CW / 8; ++c8) {
          const float4 ba = __ldg(bb + 2 * c8), bc = __ldg(bb + 2 * c8 + 1);
          const float* x8 = v + 8 * c8;
          const float2 g0 = tc::gelu2_erf_fast(tc::add2(make_float2(x8[0], x8[1]), make_float2(ba.x, ba.y)));
          const float2 g1 = tc::gelu2_erf_fast(tc::add2(make_float2(x8[2], x8[3]), make_float2(ba.z, ba.w)));
          const float2 g2 = tc::gelu2_erf_fast(tc::add2(make_float2(x8[4], x8[5]), make_float2(bc.x, bc.y)));
          const float2 g3 = tc::gelu2_erf_fast(tc::add2(make_float2(x8[6], x8[7]), make_float2(bc.z, bc.w)));
          hv[4 * c8 + 0] = tc::pack_bf16(g0.x, g0.y);
          hv[4 * c8 + 1] = tc::pack_bf16(g1.x, g1.y);
          hv[4 * c8 + 2] = tc::pack_bf16(g2.x, g2.y);
          hv[4 * c8 + 3] = tc::pack_bf16(g3.x, g3.y);
        }
        if (h == 0 && tl_ > 0) {   // H buffers staged the previous tile's residual reduce
          if (issuer) tc::bulk_wait_read<0>();
          asm volatile("bar.sync 1, %0;" ::"r"(ET) : "memory");
        }
#pragma unroll
        for (int c8 = 0; c8 < CW / 8; ++c8)
          *reinterpret_cast<uint4*>(hrow + (((u0 + c8) ^ (r & 7)) << 4)) =
              make_uint4(hv[4 * c8], hv[4 * c8 + 1], hv[4 * c8 + 2], hv[4 * c8 + 3]);
        tc::fence_proxy_async_smem();
        tc::mbar_arrive(&h_full[buf]);
        if (st) MTL(1, gc, 3);
      }
      // O^T -> residual stream: thread = feature f (TMEM lane), columns = tokens.
      if (warp == 4 && lane == 0) MTL(1, tl_ * NCH + 7, 4);
      tc::mbar_wait(o_full, tl_ & 1);
      if (warp == 4 && lane == 0) MTL(1, tl_ * NCH + 7, 5);
      tc::tc_fence_after();
      // warpgroup wg: feature half (wg & 1) on TMEM lanes, token sub-range (wg >> 1)
      constexpr int TPW = 32 / (EW / 2);   // tokens per warpgroup per 32-token group
      const int f = (wg & 1) * 128 + r;
      const int tsub = (wg >> 1) * TPW;
      const float bf = __ldg(b2 + f);
      // O^T (+ b_2) -> shared staging [32 tokens][256 features] fp32 in the two H
      // buffers (free once o_full fired), then one bulk reduce-add per 32 tokens
      // into the contiguous z rows (cp.reduce.async.bulk .add.f32: the L2 does the
      // read-modify-write, asynchronously).  One add per element: deterministic.
#pragma unroll 1
      for (int c0 = 0; c0 < BM; c0 += 32) {
        uint32_t o[TPW];
        if constexpr (TPW == 32)
          tc::tmem_ld32(lane_addr + 256 + (wg & 1) * 128 + c0, *reinterpret_cast<uint32_t(*)[32]>(o));
        else
          tc::tmem_ld16(lane_addr + 256 + (wg & 1) * 128 + c0 + tsub, *reinterpret_cast<uint32_t(*)[16]>(o));
        tc::tmem_ld_wait();
        if (c0 == BM - 32) {
          tc::tc_fence_before();
          tc::mbar_arrive(o_free);
        }
        const int64_t t0 = tile * BM + c0;
        if (t0 >= M) continue;   // CTA-uniform; groups past the end are neither staged nor issued
        float* stg = reinterpret_cast<float*>(sH + ((c0 >> 5) & 1) * H_BYTES);
        if (c0 >= 64) {   // staging buffer reused: the reduce issued two groups ago has read it
          if (issuer) tc::bulk_wait_read<1>();
          asm volatile("bar.sync 1, %0;" ::"r"(ET) : "memory");
        }
#pragma unroll
        for (int j = 0; j < TPW; ++j) stg[(tsub + j) * DM + f] = __uint_as_float(o[j]) + bf;
        tc::fence_proxy_async_smem();
        asm volatile("bar.sync 1, %0;" ::"r"(ET) : "memory");
        if (issuer) {
          const uint32_t bytes = (uint32_t)((M - t0 < 32 ? M - t0 : 32) * DM * 4);
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                       ::"l"(z + t0 * DM), "r"(tc::smem_u32(stg)), "r"(bytes) : "memory");
          tc::bulk_commit();
        }
      }
      if (warp == 4 && lane == 0) MTL(1, tl_ * NCH + 7, 6);
    }
  }
  if (warp == 4 && lane == 0) tc::bulk_wait_all();   // residual reductions complete before exit
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc::tc_fence_after();
    tc::tmem_dealloc(tmem, 512);
  }
}

}  // namespace

bool launch_mlp_fused(const void* xn, int64_t rows_alloc, const void* w1, const float* b1, const void* w2,
                      const float* b2, float* z, int64_t M, int D, cudaStream_t st) {
  if (D != DM || M <= 0) return false;
  CUtensorMap tx, t1, t2;
  if (!make_tmap_bf16(&tx, xn, rows_alloc, DM, DM, BM, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&t1, w1, FH, DM, DM, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&t2, w2, DM, FH, FH, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess)
      return false;
    attr = true;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tiles = (M + BM - 1) / BM;
  const int grid = (int)std::min<int64_t>(tiles, sms);
  mlp_tc_kernel<<<grid, THREADS, SMEM, st>>>(tx, t1, t2, b1, b2, z, M, g_mlp_timeline);
  return true;
}

}  // namespace orbit2
