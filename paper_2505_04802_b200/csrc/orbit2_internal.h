// orbit2_internal.h -- internal definitions shared by the planner, the ABI
// layer and the kernels of liborbit2.so.  Not part of the public ABI.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/orbit2.h"

namespace orbit2 {

constexpr int kQBlock = 128;       // attention query/key block (tcgen05 M = 128)
constexpr int kAlign = 1024;       // workspace region alignment (SW128 atoms)

inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

// One rank-local tile as the kernels see it (uploaded into the workspace).
struct DevTile {
  int32_t pad_y0, pad_x0, pad_h, pad_w;      // padded rect (patch units)
  int32_t core_y0, core_x0, core_h, core_w;  // core rect (patch units)
  int32_t n_tokens, n_core;                   // n_core: tokens with decoder outputs (= core tokens
                                              // unless dec_hidden > 0: core + ring, R32)
  int32_t qb_off;                             // first query block (local numbering)
  int32_t qp_off;                             // first query-block PAIR (local numbering)
  int64_t tok_off;                            // token offset in local packing (one sample)
  int64_t core_off;                           // offset of the tile's output tokens in the output packing
  int32_t out_y0, out_x0, out_h, out_w;       // output-token rect (patch units): the core grown by
                                              // ceil(2/P) patches when dec_hidden > 0, clipped to the grid
};
static_assert(sizeof(DevTile) == 80, "DevTile layout");

// Per-call geometry of a chunk of rank-local tiles [tb, tb+tc) for B samples.
struct Chunk {
  int32_t tb, tc;
  int64_t tok0, core0;        // local offsets of the first tile
  int64_t chunk_tokens;       // tokens per sample in this chunk
  int64_t chunk_core;         // core tokens per sample in this chunk
  int32_t qb0, nqb;           // query blocks (per sample) of the chunk
  int32_t qp0, nqp;           // query-block pairs (per sample) of the chunk
  int32_t qc0, nqc;           // last block: query-block pairs holding core tokens (per sample)
  int32_t qg0, nqg, qgc0, nqgc;  // groups of 3 query blocks: all / holding core tokens (per sample)
};

// Byte offsets of the workspace regions (from the workspace base).
struct Layout {
  int64_t rowinfo, patches, z, xn, qkv, ao, hid, hin;
  int64_t tiles, qblk_tile, qpair_tile, qpair_core, core_row, pos_u, pos_w, cmap, peer_tiles, rects;
  int64_t qg3, qg3c;
  int64_t core_rblk;          // last block: 128-row blocks holding core tokens (unchunked call)
  int64_t sig, push, sigtab;  // peer-memory SP: barrier flags, push table, peers' flag pointers
  int64_t rconv, dconv;       // residual / decoder convolution weights (fp32; staged by prepare_weights)
  int64_t total;
  int64_t mrow, mcore;        // rows of the token and core-token buffers
  int32_t din_pad;            // K of the embedding GEMM: round_up(Din, 64)
  int32_t ld_patch;           // row stride of TMA-gathered bf16 patch rows: round_up(Din, 8)
  int32_t k_agg_pad;          // R33: K of the aggregation GEMM (round_up(H V (p^2 + 1), 64)); 0 = off
  int64_t agg;                // R33: aggregation A-operand rows [rows][k_agg_pad]
  int32_t esize;              // activation element size (2 bf16, 4 fp32)
};

// A rectangle of coarse pixels with its element offset in a transfer message.
struct DevRect {
  int32_t y0, y1, x0, x1;
  int64_t off;      // first element (floats) of this rect in the message: [B][V][rows][cols]
  int64_t pad_;
};
static_assert(sizeof(DevRect) == 32, "DevRect layout");

struct XferList {   // one (kind, peer, direction) list inside the workspace rect table
  int32_t start, count;
  int64_t elems;
};

struct Plan {
  orbit2_config cfg;
  std::vector<int32_t> cmap;            // K entries
  std::vector<orbit2_tile> tiles;       // all tiles, tile_id order
  std::vector<int32_t> local;           // tile ids owned by cfg.rank, increasing
  std::vector<DevTile> dev;             // rank-local device table
  std::vector<int32_t> qblk_tile;       // local q-block -> local tile index
  std::vector<int32_t> qpair_tile;      // local q-block pair -> local tile index
  // last block (R16): only query pairs that hold core tokens are computed;
  // entry = local tile index << 16 | first query block << 1 | (blocks - 1)
  std::vector<int32_t> qpair_core;
  std::vector<int32_t> qpc_off;         // per local tile (+ sentinel): first qpair_core entry
  // groups of 3 query blocks (attention at head dim 64: three Q tiles share each
  // 64-key K/V block); entry = local tile << 16 | first block << 2 | (blocks - 1)
  std::vector<int32_t> qg3, qg3_off;    // every group; per local tile (+ sentinel) first entry
  std::vector<int32_t> qg3c, qg3c_off;  // last block: groups holding core tokens
  std::vector<int32_t> core_row;        // local core token -> local padded token index
  // last block (R16) of a call over every rank-local tile (all B samples): the
  // 128-row blocks of the packed token rows that hold core tokens (block tail)
  std::vector<int32_t> core_rblk;
  orbit2_plan_info info;
  Layout lay;
  int32_t Hp, Wp, P, D, d, Din, Nh, max_pad_h, max_pad_w, max_core_h, max_core_w;
  int32_t k_agg = 0;                    // R33: H V (p^2 + 1)
  // multi-rank: every rank's device tile table (for orbit2_stitch_peer) and
  // this rank's transfer rectangle lists
  std::vector<std::vector<DevTile>> dev_by_rank;   // with sentinel
  std::vector<int64_t> peer_tab_off;               // element offset of rank r's table in peer_tiles
  std::vector<int64_t> local_core_by_rank;
  std::vector<DevRect> rects;                      // all lists back to back
  std::vector<XferList> xfer;                      // index ((kind * R) + peer) * 2 + direction
  int32_t n_push = 0;                              // HALO SEND rectangles over all peers
};
// One halo-push rectangle (coarse pixels) with the peer's input field it goes to.
struct DevPush {
  int32_t y0, y1, x0, x1;
  float* dst;       // the peer's input field [B][V][H][W], mapped into this process
  int64_t pad_;
};
static_assert(sizeof(DevPush) == 32, "DevPush layout");

// rectangles of one transfer (host side, pure)
void xfer_rects(const Plan& p, int kind, int rank, int peer, int direction, std::vector<orbit2_rect>* out);

// planner (plan.cpp); returns status and fills msg on error
orbit2_status build_plan(const orbit2_config* cfg, Plan* plan, std::string* msg);
Chunk make_chunk(const Plan& plan, int32_t tb, int32_t tc);

// Packed-weight offsets (bytes from the packed base).
struct LayerW {
  int64_t ln1_g, ln1_b, w_qkv, b_qkv, w_o, b_o, ln2_g, ln2_b, w_1, b_1, w_2, b_2;
};
struct WeightLayout {
  int64_t w_e, bias_e, lnf_g, lnf_b, w_h, b_h;
  int64_t rconv, dconv;       // residual / decoder convolution weights (fp32 copies of the canonical tail)
  int64_t agg_b, agg_w, agg_c;  // R33 fused aggregation: GEMM B [D][k_agg_pad], score weights, score offsets
  std::vector<LayerW> layers;
  int64_t total;
  // canonical (fp32 element) offsets, same names
  int64_t c_w_e, c_b_e, c_e_s, c_lnf_g, c_lnf_b, c_w_h, c_b_h, c_rconv, c_dconv, c_agg;
  std::vector<LayerW> c_layers;
  int64_t c_total;
};
WeightLayout weight_layout(const Plan& plan);

}  // namespace orbit2
