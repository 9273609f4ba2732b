// plan.cpp -- step (1) planning of the TILES pass: tile rectangles, halo,
// packing offsets, rank assignment, analytic counts and the workspace layout.
// Host-only, pure, no CUDA.
//
// P:527 "TILES partitions both inputs and downscaled outputs into spatial
// tiles"; "each tile is extended with a fixed-width halo ... that
// overlaps adjacent tiles".  Readings: R3 halo in patches, R4
// CLAMP at the grid border (REPLICATE optional), R5 earlier tiles take the
// remainder, R6 row-major tile ids and token order.
#include <algorithm>
#include <cstdio>
#include <numeric>

#include "orbit2_internal.h"

namespace orbit2 {

namespace {

std::vector<int32_t> split(int32_t n, int32_t parts) {
  std::vector<int32_t> r(parts);
  for (int32_t i = 0; i < parts; ++i) r[i] = n / parts + (i < n % parts ? 1 : 0);
  return r;
}

bool fail(std::string* msg, const char* text) {
  if (msg) *msg = text;
  return false;
}

bool validate(const orbit2_config* c, std::string* msg, orbit2_status* st) {
  *st = ORBIT2_E_INVALID;
  if (!c) return fail(msg, "cfg: null pointer");
  if (c->abi_version != ORBIT2_ABI_VERSION) return fail(msg, "abi_version: does not match ORBIT2_ABI_VERSION");
  if (c->batch < 1) return fail(msg, "batch: must be >= 1");
  if (c->patch < 1) return fail(msg, "patch: must be >= 1");
  if (c->H < 1 || c->W < 1) return fail(msg, "H/W: must be >= 1");
  if (c->H % c->patch) return fail(msg, "H: patch does not divide H");
  if (c->W % c->patch) return fail(msg, "W: patch does not divide W");
  if (c->V < 1) return fail(msg, "V: must be >= 1");
  if (c->K < 1) return fail(msg, "K: must be >= 1");
  if (c->scale < 1) return fail(msg, "scale: must be >= 1");
  if (c->tiles_y < 1 || c->tiles_y > c->H / c->patch) return fail(msg, "tiles_y: must be in [1, H/patch]");
  if (c->tiles_x < 1 || c->tiles_x > c->W / c->patch) return fail(msg, "tiles_x: must be in [1, W/patch]");
  if (c->halo < 0) return fail(msg, "halo: must be >= 0");
  if (c->halo_mode != ORBIT2_HALO_CLAMP && c->halo_mode != ORBIT2_HALO_REPLICATE)
    return fail(msg, "halo_mode: must be ORBIT2_HALO_CLAMP or ORBIT2_HALO_REPLICATE");
  if (c->embed < 4 || c->heads < 1) return fail(msg, "embed/heads: must be positive");
  if (c->embed % c->heads) return fail(msg, "embed: heads does not divide embed");
  if (c->embed % 4) return fail(msg, "embed: must be a multiple of 4 (sincos position embedding)");
  if (c->depth < 0) return fail(msg, "depth: must be >= 0");
  if (c->mlp_hidden != 4 * c->embed) return fail(msg, "mlp_hidden: must equal 4*embed");
  if (c->precision != ORBIT2_BF16 && c->precision != ORBIT2_FP32)
    return fail(msg, "precision: must be ORBIT2_BF16 or ORBIT2_FP32");
  if (c->world_size < 1 || c->rank < 0 || c->rank >= c->world_size)
    return fail(msg, "world_size/rank: need 0 <= rank < world_size");
  if (c->chunk_tiles < 0) return fail(msg, "chunk_tiles: must be >= 0");
  if (c->res_hidden < 0 || c->res_hidden > 64 || c->res_hidden % 4)
    return fail(msg, "res_hidden: must be a multiple of 4 in [0, 64]");
  if (c->dec_hidden < 0 || c->dec_hidden > 64 || c->dec_hidden % 4)
    return fail(msg, "dec_hidden: must be a multiple of 4 in [0, 64]");
  if (c->var_agg != 0 && c->var_agg != 1) return fail(msg, "var_agg: must be 0 or 1");
  if (c->var_agg && c->V > 32) return fail(msg, "V: the variable aggregation supports at most 32 variables");
  if (c->dec_hidden > 0 && c->halo < (2 + c->scale * c->patch - 1) / (c->scale * c->patch))
    return fail(msg, "halo: the decoder convolutions need halo >= ceil(2 / (scale * patch)) patches");
  if (c->out_channel_map) {
    for (int k = 0; k < c->K; ++k)
      if (c->out_channel_map[k] < 0 || c->out_channel_map[k] >= c->V)
        return fail(msg, "out_channel_map: entry outside [0, V)");
  } else if (c->K > c->V) {
    return fail(msg, "K: K > V requires out_channel_map");
  }
  int d = c->embed / c->heads;
  *st = ORBIT2_E_UNSUPPORTED;
  if (d != 32 && d != 64 && d != 128) return fail(msg, "heads: head_dim = embed/heads must be 32, 64 or 128");
  if (c->precision == ORBIT2_BF16 && c->embed % 64)
    return fail(msg, "embed: BF16 path needs embed % 64 == 0");
  if (c->precision == ORBIT2_BF16 && (int64_t)c->K * c->scale * c->patch * c->scale * c->patch % 8)
    return fail(msg, "K: BF16 path needs K * (scale * patch)^2 % 8 == 0 (16-byte head-output rows for the TMA store)");
  *st = ORBIT2_OK;
  return true;
}

}  // namespace

orbit2_status build_plan(const orbit2_config* cfg, Plan* pl, std::string* msg) {
  orbit2_status st;
  if (!validate(cfg, msg, &st)) return st;
  Plan& p = *pl;
  p = Plan{};
  p.cfg = *cfg;
  const orbit2_config& c = p.cfg;
  p.Hp = c.H / c.patch;
  p.Wp = c.W / c.patch;
  p.P = c.scale * c.patch;
  p.D = c.embed;
  p.d = c.embed / c.heads;
  p.Din = c.V * c.patch * c.patch;
  p.Nh = c.K * p.P * p.P;
  p.cmap.resize(c.K);
  for (int k = 0; k < c.K; ++k) p.cmap[k] = c.out_channel_map ? c.out_channel_map[k] : k;
  p.cfg.out_channel_map = nullptr;   // do not keep the caller's pointer

  // ---- tile rectangles (R5: r_i = floor(n/T) + [i < n mod T]) ----
  std::vector<int32_t> rows = split(p.Hp, c.tiles_y), cols = split(p.Wp, c.tiles_x);
  const int32_t h = c.halo;
  int64_t tok = 0, core = 0;
  int32_t y0 = 0;
  for (int32_t i = 0; i < c.tiles_y; ++i) {
    int32_t x0 = 0;
    for (int32_t j = 0; j < c.tiles_x; ++j) {
      orbit2_tile t{};
      t.tile_id = i * c.tiles_x + j;
      t.tile_y = i;
      t.tile_x = j;
      t.core_y0 = y0; t.core_y1 = y0 + rows[i];
      t.core_x0 = x0; t.core_x1 = x0 + cols[j];
      if (c.halo_mode == ORBIT2_HALO_CLAMP) {
        t.pad_y0 = std::max(0, t.core_y0 - h); t.pad_y1 = std::min(p.Hp, t.core_y1 + h);
        t.pad_x0 = std::max(0, t.core_x0 - h); t.pad_x1 = std::min(p.Wp, t.core_x1 + h);
      } else {
        t.pad_y0 = t.core_y0 - h; t.pad_y1 = t.core_y1 + h;
        t.pad_x0 = t.core_x0 - h; t.pad_x1 = t.core_x1 + h;
      }
      t.n_tokens = (t.pad_y1 - t.pad_y0) * (t.pad_x1 - t.pad_x0);
      t.n_core_tokens = rows[i] * cols[j];
      t.token_offset = tok;
      t.core_token_offset = core;
      tok += t.n_tokens;
      core += t.n_core_tokens;
      p.tiles.push_back(t);
      x0 += cols[j];
    }
    y0 += rows[i];
  }
  const int T = (int)p.tiles.size();
  const double D = p.D, L = c.depth;
  // output tokens of a tile (R32): the core, grown by ceil(2/P) patches when the decoder
  // convolutions need the ViT output around it, clipped to the grid
  const int32_t ring = c.dec_hidden ? (2 + p.P - 1) / p.P : 0;
  auto set_out = [&](DevTile& dt) {
    dt.out_y0 = std::max(0, dt.core_y0 - ring);
    dt.out_x0 = std::max(0, dt.core_x0 - ring);
    dt.out_h = std::min(p.Hp, dt.core_y0 + dt.core_h + ring) - dt.out_y0;
    dt.out_w = std::min(p.Wp, dt.core_x0 + dt.core_w + ring) - dt.out_x0;
    dt.n_core = dt.out_h * dt.out_w;
  };
  for (orbit2_tile& t : p.tiles) {
    DevTile dt{};
    dt.core_y0 = t.core_y0; dt.core_x0 = t.core_x0;
    dt.core_h = t.core_y1 - t.core_y0; dt.core_w = t.core_x1 - t.core_x0;
    set_out(dt);
    t.n_out_tokens = dt.n_core;
  }

  // ---- rank assignment: LPT on the per-tile cost model ----
  std::vector<double> cost(T);
  for (int t = 0; t < T; ++t) {
    double n = p.tiles[t].n_tokens, cc = p.tiles[t].n_core_tokens;
    cost[t] = L * (24.0 * n * D * D + 4.0 * n * n * D) + 2.0 * cc * D * p.Nh + 2.0 * n * p.Din * D;
  }
  std::vector<int> order(T);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  std::vector<double> load(c.world_size, 0.0);
  for (int t : order) {
    int r = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    p.tiles[t].owner_rank = r;
    load[r] += cost[t];
  }
  std::vector<int32_t> nloc(c.world_size, 0);
  for (int t = 0; t < T; ++t) {
    p.tiles[t].local_index = nloc[p.tiles[t].owner_rank]++;
    if (p.tiles[t].owner_rank == c.rank) p.local.push_back(t);
  }

  // ---- rank-local device tables ----
  int64_t ltok = 0, lcore = 0;
  int32_t qb = 0, qp = 0;
  p.max_pad_h = 0;
  p.max_pad_w = 0;
  p.max_core_h = 0;
  p.max_core_w = 0;
  for (int32_t li = 0; li < (int32_t)p.local.size(); ++li) {
    const orbit2_tile& t = p.tiles[p.local[li]];
    DevTile dt{};
    dt.pad_y0 = t.pad_y0; dt.pad_x0 = t.pad_x0;
    dt.pad_h = t.pad_y1 - t.pad_y0; dt.pad_w = t.pad_x1 - t.pad_x0;
    dt.core_y0 = t.core_y0; dt.core_x0 = t.core_x0;
    dt.core_h = t.core_y1 - t.core_y0; dt.core_w = t.core_x1 - t.core_x0;
    dt.n_tokens = t.n_tokens;
    set_out(dt);
    dt.qb_off = qb;
    dt.qp_off = qp;
    dt.tok_off = ltok; dt.core_off = lcore;
    int32_t nqb = (t.n_tokens + kQBlock - 1) / kQBlock;
    for (int32_t q = 0; q < nqb; ++q) p.qblk_tile.push_back(li);
    const int32_t nqp = (nqb + 1) / 2;
    for (int32_t q = 0; q < nqp; ++q) p.qpair_tile.push_back(li);
    {   // output tokens of the tile span padded-rect tokens [c_first, c_last] (row-major)
      const int32_t c_first = (dt.out_y0 - dt.pad_y0) * dt.pad_w + (dt.out_x0 - dt.pad_x0);
      const int32_t c_last = (dt.out_y0 + dt.out_h - 1 - dt.pad_y0) * dt.pad_w + (dt.out_x0 + dt.out_w - 1 - dt.pad_x0);
      p.qpc_off.push_back((int32_t)p.qpair_core.size());
      const int32_t b0 = c_first / kQBlock, b1 = c_last / kQBlock;   // query blocks with core tokens
      if (li >= 32768 || nqb > 16384) {   // entry packing: tile index < 2^15, first block < 2^14
        if (msg) *msg = "tiles: more than 32767 tiles per rank or 16384 query blocks per tile (tile index / "
                        "block packing of the attention work lists)";
        return ORBIT2_E_UNSUPPORTED;
      }
      for (int32_t b = b0; b <= b1; b += 2)                           // entry: tile, first block, count - 1
        p.qpair_core.push_back((li << 16) | (b << 1) | (b + 1 <= b1 ? 1 : 0));
      p.qg3_off.push_back((int32_t)p.qg3.size());
      p.qg3c_off.push_back((int32_t)p.qg3c.size());
      for (int32_t b = 0; b < nqb; b += 3) p.qg3.push_back((li << 16) | (b << 2) | (std::min(3, nqb - b) - 1));
      for (int32_t b = b0; b <= b1; b += 3) p.qg3c.push_back((li << 16) | (b << 2) | (std::min(3, b1 + 1 - b) - 1));
    }
    for (int32_t u = 0; u < dt.out_h; ++u)
      for (int32_t w = 0; w < dt.out_w; ++w)
        p.core_row.push_back((int32_t)(ltok + (int64_t)(u + dt.out_y0 - dt.pad_y0) * dt.pad_w +
                                       (w + dt.out_x0 - dt.pad_x0)));
    p.max_pad_h = std::max(p.max_pad_h, dt.pad_h);
    p.max_pad_w = std::max(p.max_pad_w, dt.pad_w);
    p.max_core_h = std::max(p.max_core_h, dt.core_h);
    p.max_core_w = std::max(p.max_core_w, dt.core_w);
    qb += nqb;
    qp += nqp;
    ltok += t.n_tokens;
    lcore += dt.n_core;
    p.dev.push_back(dt);
  }
  p.qpc_off.push_back((int32_t)p.qpair_core.size());
  p.qg3_off.push_back((int32_t)p.qg3.size());
  p.qg3c_off.push_back((int32_t)p.qg3c.size());
  // sentinel entry (offsets one past the end) simplifies chunk arithmetic
  {
    DevTile end{};
    end.qb_off = qb; end.qp_off = qp; end.tok_off = ltok; end.core_off = lcore;
    p.dev.push_back(end);
  }

  // ---- every rank's tile table (output gather / stitch_peer) ----
  p.dev_by_rank.assign(c.world_size, {});
  p.local_core_by_rank.assign(c.world_size, 0);
  {
    std::vector<int64_t> rtok(c.world_size, 0), rcore(c.world_size, 0);
    for (int t = 0; t < T; ++t) {
      const orbit2_tile& tt = p.tiles[t];
      const int r = tt.owner_rank;
      DevTile dt{};
      dt.pad_y0 = tt.pad_y0; dt.pad_x0 = tt.pad_x0;
      dt.pad_h = tt.pad_y1 - tt.pad_y0; dt.pad_w = tt.pad_x1 - tt.pad_x0;
      dt.core_y0 = tt.core_y0; dt.core_x0 = tt.core_x0;
      dt.core_h = tt.core_y1 - tt.core_y0; dt.core_w = tt.core_x1 - tt.core_x0;
      dt.n_tokens = tt.n_tokens;
      set_out(dt);
      dt.tok_off = rtok[r]; dt.core_off = rcore[r];
      rtok[r] += tt.n_tokens;
      rcore[r] += dt.n_core;
      p.dev_by_rank[r].push_back(dt);
      p.max_core_h = std::max(p.max_core_h, dt.core_h);
      p.max_core_w = std::max(p.max_core_w, dt.core_w);
    }
    int64_t off = 0;
    for (int r = 0; r < c.world_size; ++r) {
      DevTile end{};
      end.tok_off = rtok[r]; end.core_off = rcore[r];
      p.dev_by_rank[r].push_back(end);
      p.local_core_by_rank[r] = rcore[r];
      p.peer_tab_off.push_back(off);
      off += (int64_t)p.dev_by_rank[r].size();
    }
  }
  // ---- this rank's transfer rectangle lists ----
  for (int kind = 0; kind < 2; ++kind)
    for (int peer = 0; peer < c.world_size; ++peer)
      for (int dir = 0; dir < 2; ++dir) {
        std::vector<orbit2_rect> rs;
        if (peer != c.rank) xfer_rects(p, kind, c.rank, peer, dir, &rs);
        XferList xl{(int32_t)p.rects.size(), (int32_t)rs.size(), 0};
        int64_t e = 0;
        for (const orbit2_rect& r : rs) {
          DevRect d{r.y0, r.y1, r.x0, r.x1, e, 0};
          p.rects.push_back(d);
          e += (int64_t)c.batch * c.V * (r.y1 - r.y0) * (r.x1 - r.x0);
        }
        xl.elems = e;
        p.xfer.push_back(xl);
      }

  // ---- last block: row blocks holding core tokens, unchunked call over all local tiles ----
  {
    const int64_t rows = (int64_t)c.batch * ltok;
    std::vector<uint8_t> need((size_t)((rows + kQBlock - 1) / kQBlock), 0);
    for (int b = 0; b < c.batch; ++b)
      for (size_t li = 0; li + 1 < p.dev.size(); ++li) {
        const DevTile& dt = p.dev[li];
        const int64_t base = (int64_t)b * ltok + dt.tok_off;
        const int64_t cf0 = (int64_t)(dt.out_y0 - dt.pad_y0) * dt.pad_w + (dt.out_x0 - dt.pad_x0);
        const int64_t cl0 = (int64_t)(dt.out_y0 + dt.out_h - 1 - dt.pad_y0) * dt.pad_w +
                            (dt.out_x0 + dt.out_w - 1 - dt.pad_x0);
        for (int64_t k = (base + cf0) / kQBlock; k <= (base + cl0) / kQBlock; ++k) need[(size_t)k] = 1;
      }
    for (size_t k = 0; k < need.size(); ++k)
      if (need[k]) p.core_rblk.push_back((int32_t)k);
  }

  // ---- info ----
  orbit2_plan_info& in = p.info;
  in = orbit2_plan_info{};
  const int32_t nl = (int32_t)p.local.size();
  in.n_tiles = T;
  in.n_local_tiles = nl;
  in.chunk_tiles = (c.chunk_tiles == 0 || c.chunk_tiles > nl) ? nl : c.chunk_tiles;
  in.head_dim = p.d;
  in.tokens_per_sample = tok;
  in.core_tokens_per_sample = core;
  in.local_tokens = ltok;
  in.local_core_tokens = lcore;
  for (int32_t a = 0; a + in.chunk_tiles <= nl || (a == 0 && nl == 0); ++a) {
    if (nl == 0) break;
    int32_t b = a + in.chunk_tiles;
    in.max_chunk_tokens = std::max<int64_t>(in.max_chunk_tokens, p.dev[b].tok_off - p.dev[a].tok_off);
    in.max_chunk_core_tokens = std::max<int64_t>(in.max_chunk_core_tokens, p.dev[b].core_off - p.dev[a].core_off);
  }
  // counts / FLOPs (SURVEY.md §8(d) formula)
  auto flops_of = [&](const std::vector<int>& ids, double* n2out, double* ncout) {
    double npad = 0, ncore = 0, n2 = 0, nc = 0;
    for (int t : ids) {
      double n = p.tiles[t].n_tokens, cc = p.tiles[t].n_core_tokens;
      npad += n; ncore += cc; n2 += n * n; nc += n * cc;
    }
    if (n2out) *n2out = n2;
    if (ncout) *ncout = nc;
    double f = 2.0 * npad * p.Din * D + 2.0 * ncore * D * p.Nh;
    if (c.depth >= 1)
      f += (L - 1) * (24.0 * npad * D * D + 4.0 * D * n2) + 4.0 * npad * D * D + 20.0 * ncore * D * D +
           4.0 * D * nc;
    return f;
  };
  std::vector<int> all(T);
  std::iota(all.begin(), all.end(), 0);
  double n2 = 0, nc = 0;
  in.flops_per_sample = flops_of(all, &n2, &nc);
  in.sum_n2_per_sample = (int64_t)n2;
  in.sum_nc_per_sample = (int64_t)nc;
  std::vector<int> loc(p.local.begin(), p.local.end());
  in.local_flops_per_sample = flops_of(loc, nullptr, nullptr);
  const double sH = (double)c.scale * c.H, sW = (double)c.scale * c.W;
  const int esz_out = c.precision == ORBIT2_BF16 ? 2 : 4;
  in.gather_bytes_per_sample = 4.0 * c.V * c.H * c.W + (double)esz_out * tok * p.Din;
  in.stitch_bytes_per_sample = (double)esz_out * c.K * sH * sW + 4.0 * c.K * c.H * c.W + 4.0 * c.K * sH * sW;
  in.canonical_weight_count = (int64_t)p.Din * p.D + 2LL * p.D +
                              (int64_t)c.depth * (12LL * p.D * p.D + 13LL * p.D) + 2LL * p.D +
                              (int64_t)p.D * p.Nh + p.Nh +
                              (c.res_hidden ? 18LL * c.res_hidden * c.K + c.res_hidden + c.K : 0) +
                              (c.dec_hidden ? 18LL * c.dec_hidden * c.K + c.dec_hidden + c.K : 0) +
                              (c.var_agg ? (int64_t)c.V * p.D * c.patch * c.patch + (int64_t)c.V * p.D + p.D +
                                               3LL * ((int64_t)p.D * p.D + p.D) : 0);
  if (c.var_agg) {   // R33: the aggregation replaces the joint embedding (2 Din D per token):
    // tokenize + key/value projections + scores + weighted sum + output projection
    const double Vd = c.V, pp = (double)c.patch * c.patch;
    const double per_tok = 2.0 * Vd * pp * D + 4.0 * Vd * D * D + 4.0 * Vd * D + 2.0 * D * D - 2.0 * p.Din * D;
    in.flops_per_sample += per_tok * (double)tok;
    in.local_flops_per_sample += per_tok * (double)ltok;
  }
  {   // the 3x3 convolution pairs on every output pixel (R31 residual, R32 decoder)
    const double cc = (double)c.res_hidden + c.dec_hidden;
    double lc = 0;
    for (int t : p.local) lc += p.tiles[t].n_core_tokens;
    in.flops_per_sample += 36.0 * c.K * cc * sH * sW;
    in.local_flops_per_sample += 36.0 * c.K * cc * lc * p.P * p.P;
  }

  // ---- workspace layout ----
  Layout& ly = p.lay;
  ly.esize = c.precision == ORBIT2_BF16 ? 2 : 4;
  ly.din_pad = (int32_t)round_up(p.Din, 64);
  // R33 aggregation as one GEMM: A row = [alpha_{h,v} a_v (H V p^2) | alpha_{h,v} (H V)], K padded to 64
  p.k_agg = c.var_agg ? c.heads * c.V * (c.patch * c.patch + 1) : 0;
  ly.k_agg_pad = c.var_agg ? (int32_t)round_up(p.k_agg, 64) : 0;
  ly.ld_patch = (int32_t)round_up(p.Din, 8);
  ly.mrow = round_up(std::max<int64_t>(1, (int64_t)c.batch * in.max_chunk_tokens), kQBlock);
  ly.mcore = round_up(std::max<int64_t>(1, (int64_t)c.batch * in.max_chunk_core_tokens), kQBlock);
  int64_t off = 0;
  auto take = [&](int64_t bytes) { int64_t o = off; off = round_up(off + std::max<int64_t>(bytes, 1), kAlign); return o; };
  const int64_t E = ly.esize;
  // peer-memory SP barrier flags [2][R] u64 + error word FIRST: peers address this
  // region in each other's workspaces, so its offset must not depend on the rank
  ly.sig = take(2LL * c.world_size * 8 + 64);
  ly.rowinfo = take(ly.mrow * 8);
  ly.patches = take(ly.mrow * ly.din_pad * E);
  ly.agg = take(c.var_agg ? ly.mrow * ly.k_agg_pad * E : 0);
  ly.z = take(ly.mrow * (int64_t)p.D * 4);
  ly.xn = take(ly.mrow * (int64_t)p.D * E);
  ly.qkv = take(ly.mrow * 3LL * p.D * E);
  ly.ao = take(ly.mrow * (int64_t)p.D * E);
  ly.hid = take(ly.mrow * 4LL * p.D * E);
  ly.hin = take(ly.mcore * (int64_t)p.D * E);
  ly.tiles = take((int64_t)p.dev.size() * sizeof(DevTile));
  ly.qblk_tile = take((int64_t)p.qblk_tile.size() * 4);
  ly.qpair_tile = take((int64_t)p.qpair_tile.size() * 4);
  ly.qpair_core = take((int64_t)p.qpair_core.size() * 4);
  ly.qg3 = take((int64_t)p.qg3.size() * 4);
  ly.qg3c = take((int64_t)p.qg3c.size() * 4);
  ly.core_rblk = take((ly.mrow / kQBlock + 1) * 4);
  ly.core_row = take((int64_t)p.core_row.size() * 4);
  ly.pos_u = take((int64_t)(p.Hp + 2 * h) * (p.D / 2) * 4);
  ly.pos_w = take((int64_t)(p.Wp + 2 * h) * (p.D / 2) * 4);
  ly.cmap = take((int64_t)c.K * 4);
  {
    int64_t n = 0;
    for (auto& v : p.dev_by_rank) n += (int64_t)v.size();
    ly.peer_tiles = take(n * (int64_t)sizeof(DevTile));
  }
  ly.rects = take((int64_t)p.rects.size() * (int64_t)sizeof(DevRect));
  // peer-memory SP (orbit2_comm_*): the push table (one entry per HALO SEND
  // rectangle of every peer) and the peers' signal pointers
  {
    int64_t n = 0;
    for (int peer = 0; peer < c.world_size; ++peer) n += p.xfer[((size_t)ORBIT2_XFER_HALO * c.world_size + peer) * 2 + ORBIT2_SEND].count;
    ly.push = take(n * 32);
    p.n_push = (int32_t)n;
  }
  ly.sigtab = take((int64_t)c.world_size * 8);
  // residual convolution weights, staged by orbit2_prepare_weights for orbit2_stitch
  ly.rconv = take(c.res_hidden ? (18LL * c.res_hidden * c.K + c.res_hidden + c.K) * 4 : 0);
  ly.dconv = take(c.dec_hidden ? (18LL * c.dec_hidden * c.K + c.dec_hidden + c.K) * 4 : 0);
  ly.total = off;
  in.workspace_bytes = ly.total;
  in.tile_out_bytes = (int64_t)c.batch * in.max_chunk_core_tokens * p.Nh * E;
  in.out_bytes = (int64_t)c.batch * c.K * (int64_t)(c.scale * c.H) * (int64_t)(c.scale * c.W) * 4;
  WeightLayout wl = weight_layout(p);
  in.packed_weight_bytes = wl.total;
  return ORBIT2_OK;
}

// Transfer rectangles in coarse pixels (see include/orbit2.h, orbit2_xfer_plan).
namespace {
orbit2_rect core_px(const orbit2_tile& t, int p) {
  return {t.core_y0 * p, t.core_y1 * p, t.core_x0 * p, t.core_x1 * p};
}
// The pixels a rank needs for one of its tiles: the padded rectangle the gather
// reads (clamped to the grid, R4) and the 1-pixel support of the bilinear
// residual around the core (O7: y1 = y0 + 1) that the stitch reads -- the
// bounding box of both (they are nested: equal to the padded rect when h >= 1).
orbit2_rect pad_px(const orbit2_tile& t, int p, int H, int W, int dil) {
  return {std::max(0, std::min(t.pad_y0 * p, t.core_y0 * p - dil)), std::min(H, std::max(t.pad_y1 * p, t.core_y1 * p + dil)),
          std::max(0, std::min(t.pad_x0 * p, t.core_x0 * p - dil)), std::min(W, std::max(t.pad_x1 * p, t.core_x1 * p + dil))};
}
bool intersect(const orbit2_rect& a, const orbit2_rect& b, orbit2_rect* o) {
  o->y0 = std::max(a.y0, b.y0); o->y1 = std::min(a.y1, b.y1);
  o->x0 = std::max(a.x0, b.x0); o->x1 = std::min(a.x1, b.x1);
  return o->y0 < o->y1 && o->x0 < o->x1;
}
}  // namespace

void xfer_rects(const Plan& p, int kind, int rank, int peer, int direction, std::vector<orbit2_rect>* out) {
  out->clear();
  const int pp = p.cfg.patch, H = p.cfg.H, W = p.cfg.W;
  // direction RECV of (rank <- peer) equals direction SEND of (peer -> rank)
  const int dst = direction == ORBIT2_RECV ? rank : peer;
  const int src = direction == ORBIT2_RECV ? peer : rank;
  if (kind == ORBIT2_XFER_CORES) {   // src's owned cores
    for (const orbit2_tile& t : p.tiles)
      if (t.owner_rank == src) out->push_back(core_px(t, pp));
    return;
  }
  for (const orbit2_tile& t : p.tiles) {          // dst's padded rects
    if (t.owner_rank != dst) continue;
    // bilinear support: 1 coarse pixel; with the residual convolutions (R31) their
    // 2-output-pixel receptive field adds ceil(2 / s) coarse pixels
    const int dil = 1 + (p.cfg.res_hidden ? (2 + p.cfg.scale - 1) / p.cfg.scale : 0);
    const orbit2_rect need = pad_px(t, pp, H, W, dil);
    for (const orbit2_tile& u : p.tiles) {        // src's cores
      if (u.owner_rank != src) continue;
      orbit2_rect o;
      if (!intersect(need, core_px(u, pp), &o)) continue;
      bool dup = false;
      for (const orbit2_rect& r : *out)
        if (r.y0 == o.y0 && r.y1 == o.y1 && r.x0 == o.x0 && r.x1 == o.x1) dup = true;
      if (!dup) out->push_back(o);
    }
  }
}

Chunk make_chunk(const Plan& p, int32_t tb, int32_t tc) {
  Chunk ch{};
  ch.tb = tb;
  ch.tc = tc;
  ch.tok0 = p.dev[tb].tok_off;
  ch.core0 = p.dev[tb].core_off;
  ch.chunk_tokens = p.dev[tb + tc].tok_off - ch.tok0;
  ch.chunk_core = p.dev[tb + tc].core_off - ch.core0;
  ch.qb0 = p.dev[tb].qb_off;
  ch.nqb = p.dev[tb + tc].qb_off - ch.qb0;
  ch.qp0 = p.dev[tb].qp_off;
  ch.nqp = p.dev[tb + tc].qp_off - ch.qp0;
  ch.qc0 = p.qpc_off[tb];
  ch.nqc = p.qpc_off[tb + tc] - ch.qc0;
  ch.qg0 = p.qg3_off[tb];
  ch.nqg = p.qg3_off[tb + tc] - ch.qg0;
  ch.qgc0 = p.qg3c_off[tb];
  ch.nqgc = p.qg3c_off[tb + tc] - ch.qgc0;
  return ch;
}

WeightLayout weight_layout(const Plan& p) {
  WeightLayout w{};
  const int64_t D = p.D, F = 4LL * p.D, Din = p.Din, Nh = p.Nh;
  const int64_t E = p.cfg.precision == ORBIT2_BF16 ? 2 : 4;
  const int64_t dinp = round_up(Din, 64);
  int64_t off = 0;
  auto take = [&](int64_t bytes) { int64_t o = off; off = round_up(off + bytes, 256); return o; };
  w.w_e = take(D * dinp * E);
  w.bias_e = take(D * 4);
  for (int l = 0; l < p.cfg.depth; ++l) {
    LayerW L{};
    L.ln1_g = take(D * 4); L.ln1_b = take(D * 4);
    L.w_qkv = take(3 * D * D * E); L.b_qkv = take(3 * D * 4);
    L.w_o = take(D * D * E); L.b_o = take(D * 4);
    L.ln2_g = take(D * 4); L.ln2_b = take(D * 4);
    L.w_1 = take(F * D * E); L.b_1 = take(F * 4);
    L.w_2 = take(D * F * E); L.b_2 = take(D * 4);
    w.layers.push_back(L);
  }
  w.lnf_g = take(D * 4); w.lnf_b = take(D * 4);
  w.w_h = take(Nh * D * E); w.b_h = take(Nh * 4);
  const int64_t CR = p.cfg.res_hidden, K = p.cfg.K;
  w.rconv = CR ? take((18 * CR * K + CR + K) * 4) : 0;   // fp32, canonical order (W_ra b_ra W_rb b_rb)
  const int64_t CD = p.cfg.dec_hidden;
  w.dconv = CD ? take((18 * CD * K + CD + K) * 4) : 0;   // fp32 (W_da b_da W_db b_db)
  // R33 fused aggregation: B operand [D][k_agg_pad] (G | E), score weights w[H V p^2] and
  // offsets c[H V] (fp32); the fused bias goes into bias_e
  const int64_t KA = p.lay.k_agg_pad, HVP = (int64_t)p.cfg.heads * p.cfg.V * p.cfg.patch * p.cfg.patch;
  w.agg_b = p.cfg.var_agg ? take(D * KA * E) : 0;
  w.agg_w = p.cfg.var_agg ? take(HVP * 4) : 0;
  w.agg_c = p.cfg.var_agg ? take((int64_t)p.cfg.heads * p.cfg.V * 4) : 0;
  w.total = off;
  // canonical fp32 element offsets (include/orbit2.h order)
  int64_t c = 0;
  auto ctake = [&](int64_t n) { int64_t o = c; c += n; return o; };
  w.c_w_e = ctake(D * Din); w.c_b_e = ctake(D); w.c_e_s = ctake(D);
  for (int l = 0; l < p.cfg.depth; ++l) {
    LayerW L{};
    L.ln1_g = ctake(D); L.ln1_b = ctake(D);
    L.w_qkv = ctake(3 * D * D); L.b_qkv = ctake(3 * D);
    L.w_o = ctake(D * D); L.b_o = ctake(D);
    L.ln2_g = ctake(D); L.ln2_b = ctake(D);
    L.w_1 = ctake(F * D); L.b_1 = ctake(F);
    L.w_2 = ctake(D * F); L.b_2 = ctake(D);
    w.c_layers.push_back(L);
  }
  w.c_lnf_g = ctake(D); w.c_lnf_b = ctake(D);
  w.c_w_h = ctake(Nh * D); w.c_b_h = ctake(Nh);
  w.c_rconv = CR ? ctake(18 * CR * K + CR + K) : 0;
  w.c_dconv = CD ? ctake(18 * CD * K + CD + K) : 0;
  const int64_t Vv = p.cfg.V, pp2 = (int64_t)p.cfg.patch * p.cfg.patch;
  w.c_agg = p.cfg.var_agg ? ctake(Vv * D * pp2 + Vv * D + D + 3 * (D * D + D)) : 0;
  w.c_total = c;
  return w;
}

}  // namespace orbit2
