// mlp_tc.cu -- fused transformer MLP on tcgen05 for D = 256 (the 9.5M-class
// Reslim):   z += W_2 . GELU(W_1 . x + b_1) + b_2      (R9, exact-erf GELU)
// with x = LN2(z) in bf16.  The 128 x 1024 hidden tile of a row block never
// leaves the SM: S_h = X W_1[h]^T lands in TMEM, 8 epilogue warps apply bias +
// GELU and write bf16 H_h BACK INTO TMEM over S_h, and the tensor core
// accumulates O += H_h W_2[:,h]^T with H_h as the TMEM A operand (TS form).
// Saves the 2 x 4D x 2 B per token hidden-activation round trip through HBM of
// the unfused pair, and H never touches shared memory (the kernel is bound by
// shared-memory bandwidth: an SS MMA with N = 128 reads 128 B/clk of operands).
//
// Persistent, one CTA per SM, warp-specialised (384 threads):
//   warp 0 lane 0 : TMA producer: X tile (64 KB) per row block, then W_1 / W_2
//                   slices (32 KB slots) through a 3-slot ring, in the order the
//                   MMA consumes them: W1(0) W1(1) W2(0) W1(2) W2(1) ... W2(7)
//   warp 1 lane 0 : MMA issuer: GEMM1(h) into S buffer h&1 (SS, N = 128; waits
//                   until GEMM2(h-2) has consumed the buffer's H), GEMM2(h-1)
//                   O[128 tokens x 256] += H W2^T (TS, N = 256)
//   warp 2        : TMEM allocator (512 columns: S/H 2 x 128, O 256)
//   warps 4-11    : epilogue, 2 warpgroups (64 hidden columns each): bias + GELU
//                   in packed f32x2 arithmetic, bf16 H into the warpgroup's own
//                   S columns; at the end of a row block O + b_2 goes through
//                   swizzled smem staging to z by TMA tensor reduce-add (the L2
//                   does the read-modify-write; one add per element:
//                   deterministic) while the warps start the next block
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>

#include <atomic>

#include "kernels.h"
#include "tc_common.cuh"

namespace orbit2 {

long long* g_mlp_timeline = nullptr;   // debug: set by orbit2_debug_mlp_timeline

bool make_tmap_bf16(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                    int box_cols, CUtensorMapSwizzle swz);
bool make_tmap_f32(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, int box_rows,
                   int box_cols, CUtensorMapSwizzle swz);

namespace {

constexpr int BM = 128;
constexpr int DM = 256;         // model width D
constexpr int FH = 1024;        // hidden width 4D
constexpr int HC = 128;         // hidden chunk
constexpr int NCH = FH / HC;    // 8 chunks
#ifndef ORBIT2_MLP_RS
#define ORBIT2_MLP_RS 3
#endif
#ifndef ORBIT2_MLP_ZC
#define ORBIT2_MLP_ZC 32
#endif
constexpr int RS = ORBIT2_MLP_RS;   // ring slots
constexpr int SLOT = 32768;
constexpr int X_BYTES = BM * DM * 2;     // 64 KB
constexpr int ZC = ORBIT2_MLP_ZC;         // residual chunk: 16 (64-byte rows, SW64) or 32 features (SW128)
constexpr int STG_BYTES = 2 * BM * ZC * 4;   // residual staging per warpgroup: 2 x (128 rows x 16 fp32)
constexpr int SMEM = X_BYTES + RS * SLOT + 2 * STG_BYTES + 1024 + 512;
constexpr int EW = 2;                    // epilogue warpgroups (4 warps each: the TMEM lane quarters)
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
                  const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmZ,
                  const float* __restrict__ b1, const float* __restrict__ b2, int64_t M,
                  long long* __restrict__ tl) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // align inside the __shared__ array (keeps the shared address space: STS, not generic ST)
  uint8_t* smem = smem_raw + ((1024u - (tc::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;
  uint8_t* sW = sX + X_BYTES;          // [RS][SLOT]
  uint8_t* sZ = sW + RS * SLOT;        // [EW][STG_BYTES] residual staging
  uint64_t* bar = reinterpret_cast<uint64_t*>(sZ + EW * STG_BYTES);
  uint64_t* x_full = bar;
  uint64_t* x_free = x_full + 1;
  uint64_t* w_full = x_free + 1;       // [RS]
  uint64_t* w_empty = w_full + RS;     // [RS]
  uint64_t* s_full = w_empty + RS;     // [2] S_h in TMEM
  uint64_t* h_full = s_full + 2;       // [2] H_h written over S_h
  uint64_t* h_free = h_full + 2;       // [2] GEMM2(h) done: the S/H buffer may take S_{h+2}
  uint64_t* o_full = h_free + 2;
  uint64_t* o_free = o_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_free + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t num_tiles = (M + BM - 1) / BM;

  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmX);
    tc::prefetch_tmap(&tmW1);
    tc::prefetch_tmap(&tmW2);
    tc::prefetch_tmap(&tmZ);
    tc::mbar_init(x_full, 1);
    tc::mbar_init(x_free, 1);
    for (int s = 0; s < RS; ++s) {
      tc::mbar_init(&w_full[s], 1);
      tc::mbar_init(&w_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tc::mbar_init(&s_full[s], 1);
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
      constexpr uint32_t id1 = tc::idesc_bf16(BM, HC, 0, 0);   // S = X W1^T: 128 tokens x 128 hidden
      constexpr uint32_t id2 = tc::idesc_bf16(BM, DM, 0, 0);   // O = H W2^T: 128 tokens x 256 features
      const uint32_t x_addr = tc::smem_u32(sX), w_addr = tc::smem_u32(sW);
      uint32_t it = 0, tl_ = 0;
      for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl_) {
        tc::mbar_wait(x_full, tl_ & 1);
        tc::tc_fence_after();
        for (int s = 0; s <= NCH; ++s) {
          if (s < NCH) {
            const uint32_t gc = tl_ * NCH + s, buf = gc & 1, use = gc >> 1;
            MTL(0, gc, 0);
            if (use >= 1) tc::mbar_wait(&h_free[buf], (use - 1) & 1);   // GEMM2(gc - 2) read H
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
              // hidden 64 k2 .. : warpgroup k2's H, bf16 pairs at S columns 64 k2 + 0..31
              const uint32_t a_tm = tmem + hb * HC + 64 * k2;
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {     // O[t, f] += H[t, hidden] W2[f, hidden]
                const uint64_t bd = tc::sdesc(w_addr + sl * SLOT + kk * 32, 16, 1024, tc::SW_128B);
                tc::mma_bf16_ts(tmem + 256, a_tm + kk * 8, bd, id2, (h | k2 | kk) != 0);
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
    // ---------------- epilogue: 2 warpgroups ----------------
    const int q = warp & 3;
    const int wg = (warp - 4) >> 2;
    const int r = q * 32 + lane;                 // row within the block = TMEM lane
    const uint32_t lane_addr = tmem + ((uint32_t)(q * 32) << 16);
    const bool issuer = q == 0 && lane == 0;     // per warpgroup: issues its residual reductions
    const uint32_t nb = 1 + wg;                  // named barrier of this warpgroup
    uint8_t* stg = sZ + wg * STG_BYTES;
    uint32_t tl_ = 0;
    for (int64_t tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++tl_) {
      for (int h = 0; h < NCH; ++h) {
        const uint32_t gc = tl_ * NCH + h, buf = gc & 1, use = gc >> 1;
        const bool st = warp == 4 && lane == 0;
        if (st) MTL(1, gc, 0);
        tc::mbar_wait(&s_full[buf], use & 1);
        if (st) MTL(1, gc, 1);
        tc::tc_fence_after();
        const uint32_t scol = lane_addr + buf * HC + wg * CW;   // this warpgroup's S (and H) columns
        float v[CW];
#pragma unroll
        for (int c = 0; c < CW; c += 32) tc::tmem_ld32(scol + c, *reinterpret_cast<uint32_t(*)[32]>(v + c));
        tc::tmem_ld_wait();
        const float4* bb = reinterpret_cast<const float4*>(b1 + h * HC + wg * CW);
        uint32_t hv[CW / 2];   // bf16 GELU outputs, packed pairs (lower hidden index in the low half)
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
        // H over this warpgroup's own (already loaded) S columns: no cross-warpgroup hazard
        tc::tmem_st32(scol, *reinterpret_cast<const uint32_t(*)[32]>(hv));
        tc::tmem_st_wait();
        tc::tc_fence_before();
        tc::mbar_arrive(&h_full[buf]);
        if (st) MTL(1, gc, 3);
      }
      // O + b_2 -> z: thread = token row; warpgroup wg: features wg*128.. in chunks of ZC,
      // double-buffered staging
      if (warp == 4 && lane == 0) MTL(1, tl_ * NCH + 7, 4);
      tc::mbar_wait(o_full, tl_ & 1);
      if (warp == 4 && lane == 0) MTL(1, tl_ * NCH + 7, 5);
      tc::tc_fence_after();
      const int32_t m0 = (int32_t)(tile * BM);
#pragma unroll 1
      for (int k = 0; k < 128 / ZC; ++k) {
        uint32_t o[ZC];
        if constexpr (ZC == 16) tc::tmem_ld16(lane_addr + 256 + wg * 128 + k * ZC, *reinterpret_cast<uint32_t(*)[16]>(o));
        else tc::tmem_ld32(lane_addr + 256 + wg * 128 + k * ZC, *reinterpret_cast<uint32_t(*)[32]>(o));
        tc::tmem_ld_wait();
        if (k == 128 / ZC - 1) {
          tc::tc_fence_before();
          tc::mbar_arrive(o_free);
        }
        uint8_t* sb = stg + (k & 1) * (BM * ZC * 4);
        if (issuer) tc::bulk_wait_read<1>();   // this half's previous reduce has read it
        asm volatile("bar.sync %0, 128;" ::"r"(nb) : "memory");
        const float4* b4 = reinterpret_cast<const float4*>(b2 + wg * 128 + k * ZC);
        uint8_t* srow = sb + r * (ZC * 4);     // SW64: unit u of row r at u ^ ((r >> 1) & 3); SW128: u ^ (r & 7)
        const int sw = ZC == 16 ? (r >> 1) & 3 : r & 7;
#pragma unroll
        for (int u = 0; u < ZC / 4; ++u) {
          const float4 bq = __ldg(b4 + u);
          *reinterpret_cast<float4*>(srow + ((u ^ sw) << 4)) =
              make_float4(__uint_as_float(o[4 * u]) + bq.x, __uint_as_float(o[4 * u + 1]) + bq.y,
                          __uint_as_float(o[4 * u + 2]) + bq.z, __uint_as_float(o[4 * u + 3]) + bq.w);
        }
        tc::fence_proxy_async_smem();
        asm volatile("bar.sync %0, 128;" ::"r"(nb) : "memory");
        if (issuer) {
          tc::tma_reduce_add_2d(&tmZ, sb, wg * 128 + k * ZC, m0);
          tc::bulk_commit();
        }
      }
      if (warp == 4 && lane == 0) MTL(1, tl_ * NCH + 7, 6);
    }
    if (issuer) tc::bulk_wait_all();   // residual reductions complete before exit
  }
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
  CUtensorMap tx, t1, t2, tz;
  if (!make_tmap_bf16(&tx, xn, rows_alloc, DM, DM, BM, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&t1, w1, FH, DM, DM, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  if (!make_tmap_bf16(&t2, w2, DM, FH, FH, 128, 64, CU_TENSOR_MAP_SWIZZLE_128B)) return false;
  // residual stream z fp32 [M][256]: 128 x 16 reduce boxes (rows past M are clipped)
  if (!make_tmap_f32(&tz, z, M, DM, DM, BM, ZC, ZC == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
    return false;
  static std::atomic<uint64_t> attr_done{0};
  if (!smem_attr_once(reinterpret_cast<const void*>(mlp_tc_kernel), SMEM, &attr_done)) return false;
  const int sms = num_sms();
  const int64_t tiles = (M + BM - 1) / BM;
  const int grid = (int)std::min<int64_t>(tiles, sms);
  mlp_tc_kernel<<<grid, THREADS, SMEM, st>>>(tx, t1, t2, tz, b1, b2, M, g_mlp_timeline);
  return true;
}

}  // namespace orbit2
