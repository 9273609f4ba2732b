// kernels.h -- launchers of the liborbit2 kernels (host side declarations).
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdint>

#include "orbit2_internal.h"

namespace orbit2 {

enum Epi : int {
  EPI_BIAS = 0,    // C[m,n] = T(acc + bias[n])
  EPI_GELU = 1,    // C[m,n] = T(gelu(acc + bias[n]))      (R9 exact-erf GELU)
  EPI_RESID = 2,   // z[m,n] += acc + bias[n]               (fp32 residual stream)
  EPI_EMBED = 3,   // z[m,n]  = acc + bias[n] + pi(u_m, w_m)  (R7, R8)
  // LayerNorm-fused forms (N == 256 == one tile's columns: whole rows in the
  // epilogue): the updated z row is written and LN(z) -> xn (bf16) as well
  EPI_RESID_LN = 4,   // z += acc + bias; xn = LN(z)     (O-projection + LN2)
  EPI_EMBED_LN = 5,   // z = acc + bias + pi; xn = LN(z) (patch embed + LN1 of block 0)
  // training backward: C[m,n] = bf16(acc * aux[m,n]), aux = GELU'(pre-activation) (bf16
  // [M][ldc], GELU' = Phi(x) + x phi(x), R9) that the training forward's EPI_GELU kept
  EPI_DGELU = 6,
};

struct EpiParams {
  int32_t M, N;
  const float* bias;       // [N]
  void* C;                 // output matrix (T or fp32 z)
  int64_t ldc;             // elements
  const int2* rowinfo;     // EMBED: global patch coords (u, w) per row
  const float* pos_u;      // EMBED: [(Hp+2h)][D/2] = [sin(u om) | cos(u om)]
  const float* pos_w;      // EMBED: [(Wp+2h)][D/2]
  int32_t pos_off;         // halo h: table row = coord + h
  int32_t half;            // D/2
  void* xn;                // *_LN: bf16 LayerNorm output [M][N]
  const float* ln_g;       // *_LN: LayerNorm gain / bias [N]
  const float* ln_b;
  // training: EPI_GELU also stores GELU'(pre-activation) (bf16, same ldc) here; EPI_RESID
  // reads the residual input from here (fp32, same ldc) instead of C (C = aux + acc + bias);
  // EPI_DGELU: the GELU' factor it multiplies by
  const void* aux = nullptr;
  int32_t single_cta = 0;  // host-side: 1 = no CTA-pair tiles (ORBIT2_SINGLE_CTA_GEMM=1, tests / A/B)
};

struct GemmOperand {
  const void* ptr;         // row-major [rows][ld] (K contiguous)
  int64_t rows;            // allocated rows (TMA extent)
  int64_t ld;              // elements per row
  int64_t cols = 0;        // valid columns (TMA extent; zero-filled up to K); 0 = K
};

// Tiles/chunk view for the token-level kernels.
struct ChunkDev {
  const DevTile* tiles;    // local table (with sentinel)
  int32_t tb, tc;
  int64_t tok0, core0, chunk_tokens, chunk_core;
  int32_t qb0, nqb;
  int32_t qp0, nqp;
  const int32_t* qblk_tile;
  const int32_t* qpair_tile;
  const int32_t* qpair_core;   // last block: (tile << 16 | first block << 1 | blocks - 1) holding core tokens
  int32_t qc0, nqc;
  int32_t core_pairs;          // attention over qpair_core instead of every pair
  const int32_t* qg3;          // groups of 3 query blocks (tile << 16 | first block << 2 | blocks - 1)
  const int32_t* qg3c;         // last block: groups holding core tokens
  int32_t qg0, nqg, qgc0, nqgc;
  const int32_t* core_row;
};

// ---- SIMT kernels (kernels_simt.cu) ----
template <typename T>
void launch_gather(const float* x, T* patches, int2* rowinfo, const ChunkDev& ch, int B, int V, int H,
                   int W, int p, int din, int din_pad, int max_pad_h, cudaStream_t st);
// bf16 CLAMP-mode gather with TMA-staged input boxes: patch rows of ld = round_up(din, 8)
// columns (no zero columns: the embed GEMM's TMA zero-fills K past din).  Returns
// false when the shape is outside what it handles (caller falls back to launch_gather).
bool launch_gather_tma(const float* x, __nv_bfloat16* patches, int2* rowinfo, const ChunkDev& ch, int B, int V,
                       int H, int W, int p, int din, int ld, int max_pad_h, int max_pad_w, cudaStream_t st);
// bf16 stitch for P = 8 with TMA-staged tile_out boxes and a separable residual;
// false when the shape is outside what it handles (caller falls back to launch_stitch).
bool launch_stitch_tma(const __nv_bfloat16* tile_out, int64_t tile_out_rows, const float* x, float* out,
                       const ChunkDev& ch, const int32_t* cmap, int B, int V, int H, int W, int K, int s, int P,
                       int max_core_h, int max_core_w, cudaStream_t st);
// stitch with the residual-path (R31) and / or decoder (R32) convolutions, fp32
// CUDA-core convolutions (rconv.cu); wres / wdec null when CR / CD == 0
template <typename T>
bool launch_stitch_conv(const T* tile_out, const float* x, float* out, const ChunkDev& ch, const int32_t* cmap,
                        const float* wres, const float* wdec, int B, int V, int H, int W, int K, int s, int P, int CR,
                        int CD, int max_core_h, int max_core_w, cudaStream_t st);
// R33 variable aggregation as one GEMM (varagg.cu): fused weights at prepare time,
// per-token score / softmax prologue writing the GEMM A rows
template <typename T>
bool launch_agg_prepare(const float* canon, const float* e_s, T* Bm, float* w, float* cc, float* bias, int V, int D,
                        int H, int pp, int KA, cudaStream_t st);
template <typename T>
bool launch_agg_prologue(const T* patches, int64_t ldp, T* agg, int64_t lda, const float* w, const float* cc,
                         int64_t M, int V, int H, int pp, cudaStream_t st);
bool make_tmap_f32_3d(CUtensorMap* map, const void* ptr, int64_t d0, int64_t d1, int64_t d2, int b0, int b1,
                      int b2);
template <typename T>
void launch_layernorm(const float* z, const float* g, const float* b, T* out, int64_t M, int D,
                      const ChunkDev* compact /* null = identity rows */, cudaStream_t st);
template <typename T>
void launch_stitch(const T* tile_out, const float* x, float* out, const ChunkDev& ch, const int32_t* cmap,
                   int B, int V, int H, int W, int K, int s, int P, int max_core_h, cudaStream_t st);
void launch_sgemm(int epi, const float* A, int64_t lda, const float* Bw, int64_t ldb, int64_t M, int64_t N,
                  int64_t K, const EpiParams& ep, cudaStream_t st);
void launch_attention_f32(const float* qkv, float* out, const ChunkDev& ch, int B, int D, int heads, int d,
                          cudaStream_t st);
void launch_xfer(const DevRect* rects, int count, int B, int V, int H, int W, const float* src, float* dst, int pack,
                 cudaStream_t st);
// ---- peer-memory SP (comm.cu) ----
void launch_push(const DevPush* tab, int count, int B, int V, int H, int W, const float* src, cudaStream_t st);
void launch_barrier(uint64_t* const* sigtab, int R, int me, int slot, uint64_t epoch, uint32_t* err,
                    cudaStream_t st);
// base and size of the device allocation holding p (driver cuMemGetAddressRange)
bool alloc_range(const void* p, void** base, size_t* bytes);
void launch_pos_tables(float* pos_u, float* pos_w, int Hp, int Wp, int h, int D, cudaStream_t st);
void launch_convert_rows(const float* src, void* dst, int64_t rows, int64_t cols, int64_t ld_dst, int to_bf16,
                         cudaStream_t st);
void launch_add_vec(const float* a, const float* b, float* out, int64_t n, cudaStream_t st);

// ---- tcgen05 / TMA kernels ----
// bf16 A [M][K] x bf16 B [N][K]^T, fp32 accumulate in TMEM, fused epilogue.
// Returns false if the shape is unsupported.
bool launch_gemm_tc(int epi, int out_bf16, const GemmOperand& A, const GemmOperand& Bw, int64_t M, int64_t N,
                    int64_t K, const EpiParams& ep, cudaStream_t st);
bool launch_attention_tc(const void* qkv_bf16, int64_t qkv_rows, void* out_bf16, const ChunkDev& ch, int B,
                         int D, int heads, int d, cudaStream_t st, float* lse = nullptr, int64_t ld_stat = 0);
// training: attention backward (attn_bwd_tc.cu), head dim 64.  dO [rows][D] bf16; lse / delta
// [heads][ld_stat] fp32 (log2-unit row log-sum-exp of the forward, sum_d dO O); dq_acc [rows][D]
// fp32 zeroed by the caller (atomics: c dS K); dK c and dV written into dqkv's K / V columns
bool launch_attention_bwd_tc(const void* qkv, const void* dout, int64_t rows, const float* lse, const float* delta,
                             int64_t ld_stat, float* dq_acc, void* dqkv, const ChunkDev& ch, int B, int D, int heads,
                             int d, cudaStream_t st);
// head dim 64: three Q tiles per CTA on 64-key blocks (attn3_tc.cu)
bool launch_attention3_tc(const void* qkv_bf16, int64_t qkv_rows, void* out_bf16, const ChunkDev& ch, int B, int D,
                          int heads, cudaStream_t st);

// Fused MLP for D = 256: z += W2 GELU(W1 x + b1) + b2 (hidden stays on chip).
bool launch_mlp_fused(const void* xn, int64_t rows_alloc, const void* w1, const float* b1, const void* w2,
                      const float* b2, float* z, int64_t M, int D, cudaStream_t st);

// Block tail for D = 256: z' = z + W_o o + b_o; z = z' + W2 GELU(W1 LN2(z') + b1) + b2
// (z' and the hidden tile stay on chip).
bool launch_block_tail(const void* ao, int64_t rows_alloc, const void* wo, const float* bo, const float* ln2_g,
                       const float* ln2_b, const void* w1, const float* b1, const void* w2, const float* b2,
                       float* z, int64_t M, int D, const float* ln1n_g /* null: no next-block LN1 */,
                       const float* ln1n_b, void* xn_next,
                       const int32_t* row_blocks /* null: every 128-row block */, int32_t n_row_blocks,
                       cudaStream_t st);

// training: weight gradients dW[n][k] += sum_m dY[m][n] X[m][k] (+ db[n] += sum_m dY[m][n] when
// db != null) with MN-major operands, split-K over the tokens, fp32 atomics (wgrad_tc.cu)
bool launch_wgrad_tc(const GemmOperand& dY, const GemmOperand& X, int64_t M, int N, int Kc, float* dW, int64_t ldo,
                     float* db, cudaStream_t st);

// ---- training step, SIMT / HBM-bound parts (train_simt.cu) ----
void launch_lat_weights(float* w, int sH, cudaStream_t st);
void launch_loss(const float* out, const float* truth, int B, int K, int sH, int sW, float lam, float delta, int geo,
                 const float* latw, double* loss, float* dout, cudaStream_t st);
void launch_stitch_bwd(const float* dout, __nv_bfloat16* dg, int64_t ldg, const ChunkDev& ch, int B, int K, int P,
                       int sH, int sW, cudaStream_t st);
bool launch_ln_bwd(const float* dy, int64_t ldy, const float* z, const float* g, const float* dres, float* dz,
                   __nv_bfloat16* dz_bf, int64_t M, int D, const int32_t* rowmap, int64_t map_per_b,
                   int64_t chunk_tokens, int64_t tok0, float* dgamma, float* dbeta, cudaStream_t st);
void launch_delta(const __nv_bfloat16* dO, const __nv_bfloat16* O, float* delta, int64_t M, int D, int heads,
                  int64_t ld_stat, cudaStream_t st);
void launch_dq_convert(const float* dq, __nv_bfloat16* dqkv, int64_t M, int D, cudaStream_t st);
void launch_transpose_bf16(const float* W, int n, int k, __nv_bfloat16* Wt, int64_t ld, cudaStream_t st);
void launch_adamw(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2, float eps,
                  float wd, float c1, float c2, cudaStream_t st);

// ---- adaptive spatial compression (compress.cu) ----
bool compress_taps(float sigma, float* w, int* r);
// Canny over B images [B][H][W]: lab = 2 on edge pixels (hysteresis on the host-driven loop);
// *passes = hysteresis passes over the field
void launch_canny(const float* img, float* tmp, float* tmp2, float* mag, uint8_t* dir, uint8_t* lab, unsigned* gmax,
                  int* changed, int B, int H, int W, float sigma, float low_frac, float high_frac, cudaStream_t st,
                  int* passes);
void launch_edges(const uint8_t* lab, uint8_t* e, int64_t n, cudaStream_t st);
// quad-tree leaves -> patches [n][4] (image, row, col, side) in (image, row, col) order,
// offsets[b] = first leaf of image b, *total = n (= offsets[B])
void launch_quadtree(const uint8_t* lab, int32_t* flag, int32_t* bsum, int32_t* total, int32_t* patches,
                     int32_t* offsets, int B, int H, int W, int mn, int mx, double thr, cudaStream_t st, int hr = 0,
                     int wr = 0, const int32_t* ext = nullptr /* per image [2]: real extents in min cells */);
void launch_tokenize(const float* feat, const int32_t* patches, int n, int C, int H, int W, int m, int D,
                     int levels, const float* wt, const float* bt, const float* es, float* rows, float* wext,
                     float* tok, cudaStream_t st);
void launch_detokenize(const float* tok, const int32_t* patches, int n, int B, int C, int H, int W, int m, int D,
                       const float* wd, const float* bd, const float* ws, const float* bs, float* proj, float* work,
                       float* out, cudaStream_t st);

// R41 / R42 (compression inside the forward, per (sample, tile) image i = b T + t):
// channel-mean field of the tile's z0 edge-padded to Hq x Wq, leaf tokens (mean of z0 over
// the leaf's rectangle patches + scale embedding), decompression of the per-token head output
// to the leaf's CORE patches in tile_out
void launch_cfield(const float* z0, const ChunkDev& ch, int T, int B, int D, int Hq, int Wq, float* f,
                   cudaStream_t st);
void launch_ctokens(const float* z0, const ChunkDev& ch, int T, const int32_t* leaves, int n, int D, const float* es,
                    float* tok, cudaStream_t st);
void launch_decompress(const __nv_bfloat16* g, const ChunkDev& ch, int T, const int32_t* leaves, int n, int Nh,
                       __nv_bfloat16* tile_out, cudaStream_t st);

// TMA descriptor encode via the driver entry point (no libcuda link dependency)
bool tma_available();

// Per-device launch state: SM count of the current device, and the dynamic
// shared-memory attribute of `func` set once per device (bit d of *done).
int num_sms();
bool smem_attr_once(const void* func, int bytes, std::atomic<uint64_t>* done);

}  // namespace orbit2
