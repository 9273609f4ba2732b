// orbit2_abi.cu -- the C ABI of liborbit2.so (include/orbit2.h): plan,
// create, weight packing, the forward (steps 1-3 + head) and the stitch
// (steps 4-5).  Orchestration only; every step of the path is a kernel.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "kernels.h"
#include "orbit2_internal.h"

using namespace orbit2;

namespace {

thread_local std::string g_err;

orbit2_status set_err(orbit2_status st, const std::string& msg) {
  g_err = msg;
  return st;
}

struct Timing {
  const char* name;
  cudaEvent_t a, b;
};

// Training workspace (orbit2_train_bind): activations the backward needs, kept per block,
// the backward's scratch and the transposed bf16 weights of the input-gradient GEMMs.
struct TrainLay {
  int64_t rows = 0, rows_core = 0;       // mrow, mcore of the plan
  int64_t nh_pad = 0;                    // K P^2 rounded up to 64 (GEMM K of dhin = dG W_h)
  // per block; gdash = GELU'(MLP pre-activation) (bf16), written by the MLP-up epilogue
  std::vector<int64_t> zin, xn1, qkv, ao, lse, zmid, xn2, gdash, hact;
  int64_t zfin = 0, hin = 0;
  int64_t dz = 0, dz_bf = 0, dzm = 0, dzm_bf = 0, dh = 0, dxn = 0, dao = 0, delta = 0, dq = 0, dqkv = 0;
  int64_t dg = 0, dhin = 0, latw = 0, zero = 0;
  std::vector<int64_t> wqkv_t, wo_t, w1_t, w2_t;   // per block, bf16 [in][out]
  int64_t wh_t = 0;                      // bf16 [D][nh_pad]
  int64_t total = 0;
};

struct Ctx {
  Plan plan;
  WeightLayout wl;
  uint8_t* ws = nullptr;
  int64_t launches = 0;
  bool profiling = false;
  std::vector<Timing> pending;
  std::vector<cudaEvent_t> pool;
  std::map<std::string, std::pair<int64_t, double>> acc;
  bool sync_check = false;
  bool trace = false;         // ORBIT2_TRACE=1: kernel names to stderr before each launch (hang hunting)
  bool unfused_mlp = false;   // ORBIT2_UNFUSED_MLP=1: two GEMMs instead of mlp_fused (D = 256)
  bool unfused_ln = false;    // ORBIT2_UNFUSED_LN=1: separate LayerNorm kernels after embed / O-proj
  int single_cta_gemm = 0;    // ORBIT2_SINGLE_CTA_GEMM=1: no CTA-pair GEMM tiles (bit-exactness tests)
  bool unfused_block = false; // ORBIT2_UNFUSED_BLOCK=1: O-proj(+LN2) GEMM and fused MLP as two kernels (D = 256)
  bool all_queries_last = false;  // ORBIT2_ALL_QUERIES_LAST=1: last block's attention over every query pair
  bool simt_gather = false;       // ORBIT2_SIMT_GATHER=1: smem-staged SIMT gather instead of the TMA one
  bool tma_stitch = false;        // ORBIT2_TMA_STITCH=1: TMA-staged stitch (measured slower than the SIMT one)
  // peer-memory SP (orbit2_comm_*)
  bool comm = false;
  int32_t gather_root = 0;
  float* own_input = nullptr;         // this rank's input field (the push source)
  float* target = nullptr;            // where this rank's stitch writes (root's field or its own)
  uint64_t epoch[2] = {0, 0};         // per barrier slot: 0 = after halo push, 1 = end of step
  std::vector<void*> opened;          // peer allocations opened with cudaIpcOpenMemHandle
  // training (orbit2_train_*)
  TrainLay tl;
  uint8_t* tws = nullptr;
  bool train_prepared = false;
  int64_t tl_lda_patch = 0, tl_cols_patch = 0;   // patch rows of the last training forward
  template <typename T>
  T* tat(int64_t off) const { return reinterpret_cast<T*>(tws + off); }

  template <typename T>
  T* at(int64_t off) const { return reinterpret_cast<T*>(ws + off); }
};

cudaEvent_t take_event(Ctx* c) {
  if (!c->pool.empty()) {
    cudaEvent_t e = c->pool.back();
    c->pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void drain_timings(Ctx* c) {
  for (auto& t : c->pending) {
    cudaEventSynchronize(t.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, t.a, t.b);
    auto& a = c->acc[t.name];
    a.first += 1;
    a.second += ms;
    c->pool.push_back(t.a);
    c->pool.push_back(t.b);
  }
  c->pending.clear();
}

// Launch wrapper: counts launches, optionally brackets them with events.
template <typename F>
orbit2_status run(Ctx* c, const char* name, cudaStream_t st, F&& f) {
  cudaEvent_t a = nullptr, b = nullptr;
  if (c->profiling) {
    a = take_event(c);
    b = take_event(c);
    cudaEventRecord(a, st);
  }
  if (c->trace) {
    std::fprintf(stderr, "[orbit2] launch %s\n", name);
    std::fflush(stderr);
  }
  bool ok = f();
  c->launches += 1;
  if (c->profiling) {
    cudaEventRecord(b, st);
    c->pending.push_back({name, a, b});
  }
  if (!ok) return set_err(ORBIT2_E_CUDA, std::string(name) + ": launch configuration rejected");
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string(name) + ": " + cudaGetErrorString(e));
  if (c->sync_check) {
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string(name) + " (sync check): " + cudaGetErrorString(e));
  }
  return ORBIT2_OK;
}

#define ORBIT2_TRY(x)                 \
  do {                                \
    orbit2_status _s = (x);           \
    if (_s != ORBIT2_OK) return _s;   \
  } while (0)

ChunkDev chunk_dev(const Ctx* c, const Chunk& ch) {
  const Plan& p = c->plan;
  ChunkDev d{};
  d.tiles = c->at<DevTile>(p.lay.tiles);
  d.tb = ch.tb;
  d.tc = ch.tc;
  d.tok0 = ch.tok0;
  d.core0 = ch.core0;
  d.chunk_tokens = ch.chunk_tokens;
  d.chunk_core = ch.chunk_core;
  d.qb0 = ch.qb0;
  d.nqb = ch.nqb;
  d.qp0 = ch.qp0;
  d.nqp = ch.nqp;
  d.qblk_tile = c->at<int32_t>(p.lay.qblk_tile);
  d.qpair_tile = c->at<int32_t>(p.lay.qpair_tile);
  d.qpair_core = c->at<int32_t>(p.lay.qpair_core);
  d.qc0 = ch.qc0;
  d.nqc = ch.nqc;
  d.qg3 = c->at<int32_t>(p.lay.qg3);
  d.qg3c = c->at<int32_t>(p.lay.qg3c);
  d.qg0 = ch.qg0;
  d.nqg = ch.nqg;
  d.qgc0 = ch.qgc0;
  d.nqgc = ch.nqgc;
  d.core_pairs = 0;
  d.core_row = c->at<int32_t>(p.lay.core_row);
  return d;
}

orbit2_status check_range(const Ctx* c, int32_t tb, int32_t tc) {
  const orbit2_plan_info& in = c->plan.info;
  if (tb < 0 || tc < 1 || tb + tc > in.n_local_tiles)
    return set_err(ORBIT2_E_INVALID, "tile_begin/tile_count: range outside the rank-local tile list");
  if (tc > in.chunk_tiles) return set_err(ORBIT2_E_INVALID, "tile_count: exceeds info.chunk_tiles");
  return ORBIT2_OK;
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

namespace orbit2 { extern long long* g_attn_timeline; extern long long* g_mlp_timeline; }

extern "C" {

const char* orbit2_last_error(void) { return g_err.c_str(); }

/* Debug only (not in orbit2.h): device buffer of 5*64*8 int64 that the next
 * attention launches fill with clock64 stamps of CTA 0; NULL disables. */
void orbit2_debug_attn_timeline(long long* dev_buf) { orbit2::g_attn_timeline = dev_buf; }
void orbit2_debug_mlp_timeline(long long* dev_buf) { orbit2::g_mlp_timeline = dev_buf; }

orbit2_status orbit2_tiles_plan(const orbit2_config* cfg, orbit2_tile* tiles, int32_t capacity,
                                orbit2_plan_info* info) {
  Plan p;
  std::string msg;
  orbit2_status st = build_plan(cfg, &p, &msg);
  if (st != ORBIT2_OK) return set_err(st, msg);
  if (info) *info = p.info;
  if (tiles == nullptr && capacity == 0) return ORBIT2_OK;
  if (capacity < p.info.n_tiles) return set_err(ORBIT2_E_CAPACITY, "capacity: smaller than n_tiles");
  if (!tiles) return set_err(ORBIT2_E_INVALID, "tiles: null with capacity > 0");
  std::memcpy(tiles, p.tiles.data(), sizeof(orbit2_tile) * p.tiles.size());
  return ORBIT2_OK;
}

orbit2_status orbit2_create(const orbit2_config* cfg, void* workspace_dev, size_t workspace_bytes, void** ctx) {
  if (!ctx) return set_err(ORBIT2_E_INVALID, "ctx: null");
  *ctx = nullptr;
  Ctx* c = new Ctx();
  std::string msg;
  orbit2_status st = build_plan(cfg, &c->plan, &msg);
  if (st != ORBIT2_OK) {
    delete c;
    return set_err(st, msg);
  }
  const Plan& p = c->plan;
  if (!workspace_dev || !aligned16(workspace_dev)) {
    delete c;
    return set_err(ORBIT2_E_INVALID, "workspace_dev: null or not 16-byte aligned");
  }
  if ((int64_t)workspace_bytes < p.info.workspace_bytes) {
    delete c;
    return set_err(ORBIT2_E_CAPACITY, "workspace_bytes: smaller than info.workspace_bytes");
  }
  if (p.cfg.precision == ORBIT2_BF16 && !tma_available()) {
    delete c;
    return set_err(ORBIT2_E_CUDA, "cuTensorMapEncodeTiled: driver entry point unavailable");
  }
  c->ws = reinterpret_cast<uint8_t*>(workspace_dev);
  c->wl = weight_layout(p);
  const char* sc = std::getenv("ORBIT2_SYNC_CHECK");
  c->sync_check = sc && sc[0] == '1';
  const char* tr = std::getenv("ORBIT2_TRACE");
  c->trace = tr && tr[0] == '1';
  const char* um = std::getenv("ORBIT2_UNFUSED_MLP");
  c->unfused_mlp = um && um[0] == '1';
  const char* ul = std::getenv("ORBIT2_UNFUSED_LN");
  c->unfused_ln = ul && ul[0] == '1';
  const char* sct = std::getenv("ORBIT2_SINGLE_CTA_GEMM");
  c->single_cta_gemm = sct && sct[0] == '1';
  const char* ub = std::getenv("ORBIT2_UNFUSED_BLOCK");
  c->unfused_block = ub && ub[0] == '1';
  const char* aq = std::getenv("ORBIT2_ALL_QUERIES_LAST");
  c->all_queries_last = aq && aq[0] == '1';
  const char* sg = std::getenv("ORBIT2_SIMT_GATHER");
  c->simt_gather = sg && sg[0] == '1';
  const char* ss = std::getenv("ORBIT2_TMA_STITCH");
  c->tma_stitch = ss && ss[0] == '1';
  cudaError_t e = cudaSuccess;
  e = cudaMemcpy(c->at<void>(p.lay.tiles), p.dev.data(), p.dev.size() * sizeof(DevTile), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !p.qblk_tile.empty())
    e = cudaMemcpy(c->at<void>(p.lay.qblk_tile), p.qblk_tile.data(), p.qblk_tile.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !p.qpair_tile.empty())
    e = cudaMemcpy(c->at<void>(p.lay.qpair_tile), p.qpair_tile.data(), p.qpair_tile.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !p.qg3.empty())
    e = cudaMemcpy(c->at<void>(p.lay.qg3), p.qg3.data(), p.qg3.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !p.qg3c.empty())
    e = cudaMemcpy(c->at<void>(p.lay.qg3c), p.qg3c.data(), p.qg3c.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !p.qpair_core.empty())
    e = cudaMemcpy(c->at<void>(p.lay.qpair_core), p.qpair_core.data(), p.qpair_core.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(c->at<void>(p.lay.sig), 0, 2ULL * p.cfg.world_size * 8 + 64);
  if (e == cudaSuccess && !p.core_rblk.empty())
    e = cudaMemcpy(c->at<void>(p.lay.core_rblk), p.core_rblk.data(), p.core_rblk.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !p.core_row.empty())
    e = cudaMemcpy(c->at<void>(p.lay.core_row), p.core_row.data(), p.core_row.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(c->at<void>(p.lay.cmap), p.cmap.data(), p.cmap.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    std::vector<DevTile> all;
    for (auto& v : p.dev_by_rank) all.insert(all.end(), v.begin(), v.end());
    if (!all.empty())
      e = cudaMemcpy(c->at<void>(p.lay.peer_tiles), all.data(), all.size() * sizeof(DevTile), cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && !p.rects.empty())
    e = cudaMemcpy(c->at<void>(p.lay.rects), p.rects.data(), p.rects.size() * sizeof(DevRect), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    launch_pos_tables(c->at<float>(p.lay.pos_u), c->at<float>(p.lay.pos_w), p.Hp, p.Wp, p.cfg.halo, p.D, 0);
    c->launches += 2;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
  }
  if (e != cudaSuccess) {
    delete c;
    return set_err(ORBIT2_E_CUDA, std::string("orbit2_create: ") + cudaGetErrorString(e));
  }
  *ctx = c;
  return ORBIT2_OK;
}

void orbit2_destroy(void* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return;
  for (void* p : c->opened) cudaIpcCloseMemHandle(p);
  for (auto& t : c->pending) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  for (auto e : c->pool) cudaEventDestroy(e);
  delete c;
}

int64_t orbit2_launch_count(void* ctx) { return ctx ? reinterpret_cast<Ctx*>(ctx)->launches : 0; }

orbit2_status orbit2_set_profiling(void* ctx, int32_t enable) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  drain_timings(c);
  c->acc.clear();
  c->profiling = enable != 0;
  return ORBIT2_OK;
}

int32_t orbit2_kernel_times(void* ctx, const char** names, int64_t* launches, double* ms, int32_t cap) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return 0;
  drain_timings(c);
  int32_t i = 0;
  for (auto& kv : c->acc) {
    if (i < cap) {
      if (names) names[i] = kv.first.c_str();
      if (launches) launches[i] = kv.second.first;
      if (ms) ms[i] = kv.second.second;
    }
    ++i;
  }
  return i;
}

orbit2_status orbit2_prepare_weights(void* ctx, const float* canonical_dev, void* packed_dev, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (!canonical_dev || !packed_dev || !aligned16(packed_dev))
    return set_err(ORBIT2_E_INVALID, "canonical_dev/packed_dev: null or not 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Plan& p = c->plan;
  const WeightLayout& w = c->wl;
  const int bf = p.cfg.precision == ORBIT2_BF16;
  uint8_t* pk = reinterpret_cast<uint8_t*>(packed_dev);
  const int64_t D = p.D, F = 4LL * p.D;
  auto conv = [&](int64_t coff, int64_t poff, int64_t rows, int64_t cols, int64_t ld, int to_bf) {
    return run(c, "prepare_weights", st, [&] {
      launch_convert_rows(canonical_dev + coff, pk + poff, rows, cols, ld, to_bf, st);
      return true;
    });
  };
  ORBIT2_TRY(conv(w.c_w_e, w.w_e, D, p.Din, p.lay.din_pad, bf));
  ORBIT2_TRY(run(c, "prepare_weights", st, [&] {
    launch_add_vec(canonical_dev + w.c_b_e, canonical_dev + w.c_e_s, reinterpret_cast<float*>(pk + w.bias_e), D, st);
    return true;
  }));
  for (int l = 0; l < p.cfg.depth; ++l) {
    const LayerW& C = w.c_layers[l];
    const LayerW& P = w.layers[l];
    ORBIT2_TRY(conv(C.ln1_g, P.ln1_g, 1, D, D, 0));
    ORBIT2_TRY(conv(C.ln1_b, P.ln1_b, 1, D, D, 0));
    ORBIT2_TRY(conv(C.w_qkv, P.w_qkv, 3 * D, D, D, bf));
    ORBIT2_TRY(conv(C.b_qkv, P.b_qkv, 1, 3 * D, 3 * D, 0));
    ORBIT2_TRY(conv(C.w_o, P.w_o, D, D, D, bf));
    ORBIT2_TRY(conv(C.b_o, P.b_o, 1, D, D, 0));
    ORBIT2_TRY(conv(C.ln2_g, P.ln2_g, 1, D, D, 0));
    ORBIT2_TRY(conv(C.ln2_b, P.ln2_b, 1, D, D, 0));
    ORBIT2_TRY(conv(C.w_1, P.w_1, F, D, D, bf));
    ORBIT2_TRY(conv(C.b_1, P.b_1, 1, F, F, 0));
    ORBIT2_TRY(conv(C.w_2, P.w_2, D, F, F, bf));
    ORBIT2_TRY(conv(C.b_2, P.b_2, 1, D, D, 0));
  }
  ORBIT2_TRY(conv(w.c_lnf_g, w.lnf_g, 1, D, D, 0));
  ORBIT2_TRY(conv(w.c_lnf_b, w.lnf_b, 1, D, D, 0));
  ORBIT2_TRY(conv(w.c_w_h, w.w_h, p.Nh, D, D, bf));
  ORBIT2_TRY(conv(w.c_b_h, w.b_h, 1, p.Nh, p.Nh, 0));
  if (p.cfg.var_agg) {   // R33: fold tokenizer + key / value / output projections into the GEMM weights
    const int pp = p.cfg.patch * p.cfg.patch;
    ORBIT2_TRY(run(c, "prepare_weights", st, [&] {
      float* fw = reinterpret_cast<float*>(pk + w.agg_w);
      float* fc = reinterpret_cast<float*>(pk + w.agg_c);
      float* fb = reinterpret_cast<float*>(pk + w.bias_e);
      if (bf)
        return launch_agg_prepare<__nv_bfloat16>(canonical_dev + w.c_agg, canonical_dev + w.c_e_s,
                                                 reinterpret_cast<__nv_bfloat16*>(pk + w.agg_b), fw, fc, fb,
                                                 p.cfg.V, p.D, p.cfg.heads, pp, p.lay.k_agg_pad, st);
      return launch_agg_prepare<float>(canonical_dev + w.c_agg, canonical_dev + w.c_e_s,
                                       reinterpret_cast<float*>(pk + w.agg_b), fw, fc, fb, p.cfg.V, p.D, p.cfg.heads,
                                       pp, p.lay.k_agg_pad, st);
    }));
  }
  // R31 / R32 convolutions: fp32 into the packed blob and the workspace (orbit2_stitch reads them there)
  const int32_t convs[2] = {p.cfg.res_hidden, p.cfg.dec_hidden};
  const int64_t c_off[2] = {w.c_rconv, w.c_dconv}, p_off[2] = {w.rconv, w.dconv}, ws_off[2] = {p.lay.rconv, p.lay.dconv};
  for (int i = 0; i < 2; ++i) {
    if (!convs[i]) continue;
    const int64_t n = 18LL * convs[i] * p.cfg.K + convs[i] + p.cfg.K;
    ORBIT2_TRY(conv(c_off[i], p_off[i], 1, n, n, 0));
    cudaError_t e = cudaMemcpyAsync(c->at<void>(ws_off[i]), canonical_dev + c_off[i], n * 4,
                                    cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("prepare_weights: ") + cudaGetErrorString(e));
  }
  return ORBIT2_OK;
}

orbit2_status orbit2_reslim_forward(void* ctx, const void* packed_w, const float* input_dev, int32_t tile_begin,
                                    int32_t tile_count, void* tile_out_dev, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (!packed_w || !input_dev || !tile_out_dev || !aligned16(packed_w) || !aligned16(input_dev) ||
      !aligned16(tile_out_dev))
    return set_err(ORBIT2_E_INVALID, "packed_w/input_dev/tile_out_dev: null or not 16-byte aligned");
  ORBIT2_TRY(check_range(c, tile_begin, tile_count));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Plan& p = c->plan;
  const orbit2_config& cf = p.cfg;
  const Layout& ly = p.lay;
  const WeightLayout& w = c->wl;
  const uint8_t* W8 = reinterpret_cast<const uint8_t*>(packed_w);
  auto wf = [&](int64_t off) { return reinterpret_cast<const float*>(W8 + off); };
  const Chunk ch = make_chunk(p, tile_begin, tile_count);
  const ChunkDev cd = chunk_dev(c, ch);
  const int B = cf.batch;
  const int64_t M = (int64_t)B * ch.chunk_tokens;
  const int64_t Mc = (int64_t)B * ch.chunk_core;
  const int64_t D = p.D, F = 4LL * p.D;
  const int64_t mrow = ly.mrow, mcore = ly.mcore;
  int2* rowinfo = c->at<int2>(ly.rowinfo);
  float* z = c->at<float>(ly.z);

  EpiParams emb{};
  emb.M = (int32_t)M; emb.N = (int32_t)D; emb.bias = wf(w.bias_e); emb.C = z; emb.ldc = D;
  emb.rowinfo = rowinfo; emb.pos_u = c->at<float>(ly.pos_u); emb.pos_w = c->at<float>(ly.pos_w);
  emb.pos_off = cf.halo; emb.half = (int32_t)(D / 2);

  if (cf.precision == ORBIT2_BF16) {
    typedef __nv_bfloat16 bf16;
    bf16* patches = c->at<bf16>(ly.patches);
    bf16* xn = c->at<bf16>(ly.xn);
    bf16* qkv = c->at<bf16>(ly.qkv);
    bf16* ao = c->at<bf16>(ly.ao);
    bf16* hid = c->at<bf16>(ly.hid);
    bf16* hin = c->at<bf16>(ly.hin);
    auto gemm = [&](const char* name, int epi, int out_bf, const void* A, int64_t arows, int64_t lda,
                    int64_t wo, int64_t n, int64_t k, int64_t rows, EpiParams ep, int64_t acols = 0) {
      GemmOperand a{A, arows, lda, acols}, b{W8 + wo, n, k};
      ep.M = (int32_t)rows;
      ep.N = (int32_t)n;
      return run(c, name, st, [&] {
        ep.single_cta = c->single_cta_gemm;
        return launch_gemm_tc(epi, out_bf, a, b, rows, n, k, ep, st);
      });
    };
    // step (1): TMA-staged gather (CLAMP halos) into patch rows of ld_patch columns;
    // the smem-staged SIMT gather with zero-padded rows otherwise (REPLICATE halos
    // read clamped edge pixels, which a TMA box would zero-fill)
    int64_t lda_patch = ly.din_pad, cols_patch = 0;
    if (cf.halo_mode == ORBIT2_HALO_CLAMP && !c->simt_gather) {
      bool ok = false;
      ORBIT2_TRY(run(c, "tile_gather", st, [&] {
        ok = launch_gather_tma(input_dev, patches, rowinfo, cd, B, cf.V, cf.H, cf.W, cf.patch, p.Din, ly.ld_patch,
                               p.max_pad_h, p.max_pad_w, st);
        return true;
      }));
      if (ok) {
        lda_patch = ly.ld_patch;
        cols_patch = p.Din;
      }
    }
    if (cols_patch == 0) {
      ORBIT2_TRY(run(c, "tile_gather", st, [&] {
        launch_gather<bf16>(input_dev, patches, rowinfo, cd, B, cf.V, cf.H, cf.W, cf.patch, p.Din, ly.din_pad,
                            p.max_pad_h, st);
        return true;
      }));
    }
    // Key/value blocks of the last tile may read up to 127 rows past M: keep
    // them finite (their probabilities are 0, but 0 * NaN would poison P.V).
    if (mrow > M) {
      cudaError_t e = cudaMemsetAsync(qkv + M * 3 * D, 0, (size_t)(mrow - M) * 3 * D * sizeof(bf16), st);
      if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("memset: ") + cudaGetErrorString(e));
    }
    // the embedding GEMM's A / B operands: patch rows x W_e, or (R33) the aggregation
    // rows [alpha a | alpha] x the folded [G | E]
    const void* embA = patches;
    int64_t embW = w.w_e, embK = ly.din_pad, embLd = lda_patch, embCols = cols_patch;
    if (cf.var_agg) {
      bf16* agg = c->at<bf16>(ly.agg);
      ORBIT2_TRY(run(c, "var_aggregate", st, [&] {
        return launch_agg_prologue<bf16>(patches, lda_patch, agg, ly.k_agg_pad, wf(w.agg_w), wf(w.agg_c), M, cf.V,
                                         cf.heads, cf.patch * cf.patch, st);
      }));
      embA = agg;
      embW = w.agg_b;
      embK = embLd = ly.k_agg_pad;
      embCols = 0;
    }
    // D == 256: one GEMM tile holds whole rows, so LayerNorms that follow a GEMM
    // run in its epilogue (embed -> LN1 of block 0, O-projection -> LN2)
    const bool ln_fused = D == 256 && !c->unfused_ln;
    if (ln_fused && cf.depth > 0) {
      EpiParams e = emb;
      e.xn = xn;
      e.ln_g = wf(w.layers[0].ln1_g);
      e.ln_b = wf(w.layers[0].ln1_b);
      ORBIT2_TRY(gemm("embed_gemm", EPI_EMBED_LN, 0, embA, mrow, embLd, embW, D, embK, M, e, embCols));
    } else {
      ORBIT2_TRY(gemm("embed_gemm", EPI_EMBED, 0, embA, mrow, embLd, embW, D, embK, M, emb, embCols));
    }
    for (int l = 0; l < cf.depth; ++l) {
      const LayerW& L = w.layers[l];
      // block 0's LN1 runs in the embed epilogue, later blocks' in the previous block_tail
      const bool tail_fused = D == 256 && !c->unfused_mlp && !c->unfused_ln && !c->unfused_block;
      if (!(ln_fused && l == 0) && !(tail_fused && l > 0)) {
        ORBIT2_TRY(run(c, "layernorm", st, [&] {
          launch_layernorm<bf16>(z, wf(L.ln1_g), wf(L.ln1_b), xn, M, (int)D, nullptr, st);
          return true;
        }));
      }
      EpiParams e{};
      e.bias = wf(L.b_qkv); e.C = qkv; e.ldc = 3 * D;
      ORBIT2_TRY(gemm("qkv_gemm", EPI_BIAS, 1, xn, mrow, D, L.w_qkv, 3 * D, D, M, e));
      ORBIT2_TRY(run(c, "tile_attention", st, [&] {
        // last block: only query pairs holding core tokens feed the head (R16)
        ChunkDev ca = cd;
        ca.core_pairs = l + 1 == cf.depth && !c->all_queries_last ? 1 : 0;
        return launch_attention_tc(qkv, mrow, ao, ca, B, (int)D, cf.heads, p.d, st);
      }));
      if (tail_fused) {
        // O-projection + residual + LN2 + MLP + residual (+ LN1 of the next block) in
        // one kernel (z' stays on chip)
        const bool nxt = l + 1 < cf.depth;
        const float* g1n = nxt ? wf(w.layers[l + 1].ln1_g) : nullptr;
        const float* b1n = nxt ? wf(w.layers[l + 1].ln1_b) : nullptr;
        const int32_t* rblk = nullptr;
        int32_t nrblk = 0;
        // last block: only row blocks holding core tokens (R16); the list is built by the
        // planner for a call over every rank-local tile and uploaded by orbit2_create
        if (!nxt && !c->all_queries_last && tile_begin == 0 && tile_count == p.info.n_local_tiles &&
            !p.core_rblk.empty()) {
          rblk = c->at<int32_t>(ly.core_rblk);
          nrblk = (int32_t)p.core_rblk.size();
        }
        ORBIT2_TRY(run(c, "block_tail", st, [&] {
          return launch_block_tail(ao, mrow, W8 + L.w_o, wf(L.b_o), wf(L.ln2_g), wf(L.ln2_b), W8 + L.w_1,
                                   wf(L.b_1), W8 + L.w_2, wf(L.b_2), z, M, (int)D, g1n, b1n, xn, rblk, nrblk,
                                   st);
        }));
        continue;
      }
      e = EpiParams{}; e.bias = wf(L.b_o); e.C = z; e.ldc = D;
      if (ln_fused) {
        e.xn = xn;
        e.ln_g = wf(L.ln2_g);
        e.ln_b = wf(L.ln2_b);
        ORBIT2_TRY(gemm("oproj_gemm", EPI_RESID_LN, 0, ao, mrow, D, L.w_o, D, D, M, e));
      } else {
        ORBIT2_TRY(gemm("oproj_gemm", EPI_RESID, 0, ao, mrow, D, L.w_o, D, D, M, e));
        ORBIT2_TRY(run(c, "layernorm", st, [&] {
          launch_layernorm<bf16>(z, wf(L.ln2_g), wf(L.ln2_b), xn, M, (int)D, nullptr, st);
          return true;
        }));
      }
      if (D == 256 && !c->unfused_mlp) {   // hidden tile stays on chip
        ORBIT2_TRY(run(c, "mlp_fused", st, [&] {
          return launch_mlp_fused(xn, mrow, W8 + L.w_1, wf(L.b_1), W8 + L.w_2, wf(L.b_2), z, M, (int)D, st);
        }));
      } else {
        e = EpiParams{}; e.bias = wf(L.b_1); e.C = hid; e.ldc = F;
        ORBIT2_TRY(gemm("mlp_up_gemm", EPI_GELU, 1, xn, mrow, D, L.w_1, F, D, M, e));
        e = EpiParams{}; e.bias = wf(L.b_2); e.C = z; e.ldc = D;
        ORBIT2_TRY(gemm("mlp_down_gemm", EPI_RESID, 0, hid, mrow, F, L.w_2, D, F, M, e));
      }
    }
    ORBIT2_TRY(run(c, "layernorm", st, [&] {
      launch_layernorm<bf16>(z, wf(w.lnf_g), wf(w.lnf_b), hin, Mc, (int)D, &cd, st);
      return true;
    }));
    EpiParams e{};
    e.bias = wf(w.b_h); e.C = tile_out_dev; e.ldc = p.Nh;
    ORBIT2_TRY(gemm("head_gemm", EPI_BIAS, 1, hin, mcore, D, w.w_h, p.Nh, D, Mc, e));
  } else {
    float* patches = c->at<float>(ly.patches);
    float* xn = c->at<float>(ly.xn);
    float* qkv = c->at<float>(ly.qkv);
    float* ao = c->at<float>(ly.ao);
    float* hid = c->at<float>(ly.hid);
    float* hin = c->at<float>(ly.hin);
    auto sg = [&](const char* name, int epi, const float* A, int64_t lda, int64_t wo, int64_t n, int64_t k,
                  int64_t rows, EpiParams ep) {
      ep.M = (int32_t)rows;
      ep.N = (int32_t)n;
      return run(c, name, st, [&] {
        launch_sgemm(epi, A, lda, wf(wo), k, rows, n, k, ep, st);
        return true;
      });
    };
    ORBIT2_TRY(run(c, "tile_gather", st, [&] {
      launch_gather<float>(input_dev, patches, rowinfo, cd, B, cf.V, cf.H, cf.W, cf.patch, p.Din, ly.din_pad,
                           p.max_pad_h, st);
      return true;
    }));
    if (cf.var_agg) {   // R33 (fp32 path)
      float* agg = c->at<float>(ly.agg);
      ORBIT2_TRY(run(c, "var_aggregate", st, [&] {
        return launch_agg_prologue<float>(patches, ly.din_pad, agg, ly.k_agg_pad, wf(w.agg_w), wf(w.agg_c), M, cf.V,
                                          cf.heads, cf.patch * cf.patch, st);
      }));
      ORBIT2_TRY(sg("embed_gemm", EPI_EMBED, agg, ly.k_agg_pad, w.agg_b, D, ly.k_agg_pad, M, emb));
    } else {
      ORBIT2_TRY(sg("embed_gemm", EPI_EMBED, patches, ly.din_pad, w.w_e, D, ly.din_pad, M, emb));
    }
    for (int l = 0; l < cf.depth; ++l) {
      const LayerW& L = w.layers[l];
      ORBIT2_TRY(run(c, "layernorm", st, [&] {
        launch_layernorm<float>(z, wf(L.ln1_g), wf(L.ln1_b), xn, M, (int)D, nullptr, st);
        return true;
      }));
      EpiParams e{};
      e.bias = wf(L.b_qkv); e.C = qkv; e.ldc = 3 * D;
      ORBIT2_TRY(sg("qkv_gemm", EPI_BIAS, xn, D, L.w_qkv, 3 * D, D, M, e));
      ORBIT2_TRY(run(c, "tile_attention", st, [&] {
        launch_attention_f32(qkv, ao, cd, B, (int)D, cf.heads, p.d, st);
        return true;
      }));
      e = EpiParams{}; e.bias = wf(L.b_o); e.C = z; e.ldc = D;
      ORBIT2_TRY(sg("oproj_gemm", EPI_RESID, ao, D, L.w_o, D, D, M, e));
      ORBIT2_TRY(run(c, "layernorm", st, [&] {
        launch_layernorm<float>(z, wf(L.ln2_g), wf(L.ln2_b), xn, M, (int)D, nullptr, st);
        return true;
      }));
      e = EpiParams{}; e.bias = wf(L.b_1); e.C = hid; e.ldc = F;
      ORBIT2_TRY(sg("mlp_up_gemm", EPI_GELU, xn, D, L.w_1, F, D, M, e));
      e = EpiParams{}; e.bias = wf(L.b_2); e.C = z; e.ldc = D;
      ORBIT2_TRY(sg("mlp_down_gemm", EPI_RESID, hid, F, L.w_2, D, F, M, e));
    }
    ORBIT2_TRY(run(c, "layernorm", st, [&] {
      launch_layernorm<float>(z, wf(w.lnf_g), wf(w.lnf_b), hin, Mc, (int)D, &cd, st);
      return true;
    }));
    EpiParams e{};
    e.bias = wf(w.b_h); e.C = tile_out_dev; e.ldc = p.Nh;
    ORBIT2_TRY(sg("head_gemm", EPI_BIAS, hin, D, w.w_h, p.Nh, D, Mc, e));
  }
  return ORBIT2_OK;
}

orbit2_status orbit2_xfer_plan(const orbit2_config* cfg, int32_t kind, int32_t peer, int32_t direction,
                               orbit2_rect* rects, int32_t cap, int32_t* n_rects, int64_t* n_elems) {
  Plan p;
  std::string msg;
  orbit2_status st = build_plan(cfg, &p, &msg);
  if (st != ORBIT2_OK) return set_err(st, msg);
  if (kind != ORBIT2_XFER_HALO && kind != ORBIT2_XFER_CORES) return set_err(ORBIT2_E_INVALID, "kind: unknown transfer");
  if (direction != ORBIT2_SEND && direction != ORBIT2_RECV) return set_err(ORBIT2_E_INVALID, "direction: unknown");
  if (peer < 0 || peer >= cfg->world_size || peer == cfg->rank)
    return set_err(ORBIT2_E_INVALID, "peer: must be another rank in [0, world_size)");
  std::vector<orbit2_rect> rs;
  xfer_rects(p, kind, cfg->rank, peer, direction, &rs);
  int64_t e = 0;
  for (const orbit2_rect& r : rs) e += (int64_t)cfg->batch * cfg->V * (r.y1 - r.y0) * (r.x1 - r.x0);
  if (n_rects) *n_rects = (int32_t)rs.size();
  if (n_elems) *n_elems = e;
  if (rects == nullptr && cap == 0) return ORBIT2_OK;
  if (cap < (int32_t)rs.size()) return set_err(ORBIT2_E_CAPACITY, "cap: smaller than the rectangle count");
  if (!rects) return set_err(ORBIT2_E_INVALID, "rects: null with cap > 0");
  std::memcpy(rects, rs.data(), rs.size() * sizeof(orbit2_rect));
  return ORBIT2_OK;
}

static orbit2_status xfer(void* ctx, int32_t kind, int32_t peer, const float* src, float* dst, int pack, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  const Plan& p = c->plan;
  if (kind != ORBIT2_XFER_HALO && kind != ORBIT2_XFER_CORES) return set_err(ORBIT2_E_INVALID, "kind: unknown transfer");
  if (peer < 0 || peer >= p.cfg.world_size || peer == p.cfg.rank)
    return set_err(ORBIT2_E_INVALID, "peer: must be another rank in [0, world_size)");
  if (!src || !dst) return set_err(ORBIT2_E_INVALID, "input_dev/buf_dev: null");
  const XferList& xl = p.xfer[((size_t)kind * p.cfg.world_size + peer) * 2 + (pack ? ORBIT2_SEND : ORBIT2_RECV)];
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  return run(c, pack ? "xfer_pack" : "xfer_unpack", st, [&] {
    launch_xfer(c->at<DevRect>(p.lay.rects) + xl.start, xl.count, p.cfg.batch, p.cfg.V, p.cfg.H, p.cfg.W, src, dst,
                pack, st);
    return true;
  });
}

orbit2_status orbit2_xfer_pack(void* ctx, int32_t kind, int32_t peer, const float* input_dev, float* buf_dev,
                               void* stream) {
  return xfer(ctx, kind, peer, input_dev, buf_dev, 1, stream);
}

orbit2_status orbit2_xfer_unpack(void* ctx, int32_t kind, int32_t peer, const float* buf_dev, float* input_dev,
                                 void* stream) {
  return xfer(ctx, kind, peer, buf_dev, input_dev, 0, stream);
}

orbit2_status orbit2_stitch_peer(void* ctx, int32_t peer, const void* tile_out_dev, const float* input_dev,
                                 float* out_dev, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  const Plan& p = c->plan;
  const orbit2_config& cf = p.cfg;
  if (peer < 0 || peer >= cf.world_size) return set_err(ORBIT2_E_INVALID, "peer: outside [0, world_size)");
  if (!tile_out_dev || !input_dev || !out_dev || !aligned16(tile_out_dev) || !aligned16(input_dev) ||
      !aligned16(out_dev))
    return set_err(ORBIT2_E_INVALID, "tile_out_dev/input_dev/out_dev: null or not 16-byte aligned");
  const int32_t n = (int32_t)p.dev_by_rank[peer].size() - 1;
  if (n == 0) return ORBIT2_OK;
  ChunkDev cd{};
  cd.tiles = c->at<DevTile>(p.lay.peer_tiles) + p.peer_tab_off[peer];
  cd.tb = 0;
  cd.tc = n;
  cd.chunk_core = p.local_core_by_rank[peer];
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int32_t* cmap = c->at<int32_t>(p.lay.cmap);
  return run(c, "stitch_residual", st, [&] {
    if (cf.res_hidden || cf.dec_hidden) {   // residual (R31) / decoder (R32) convolutions
      const float* wr = c->at<float>(p.lay.rconv);
      const float* wd = c->at<float>(p.lay.dconv);
      if (cf.precision == ORBIT2_BF16)
        return launch_stitch_conv<__nv_bfloat16>(reinterpret_cast<const __nv_bfloat16*>(tile_out_dev), input_dev,
                                                 out_dev, cd, cmap, wr, wd, cf.batch, cf.V, cf.H, cf.W, cf.K, cf.scale,
                                                 p.P, cf.res_hidden, cf.dec_hidden, p.max_core_h, p.max_core_w, st);
      return launch_stitch_conv<float>(reinterpret_cast<const float*>(tile_out_dev), input_dev, out_dev, cd, cmap, wr,
                                       wd, cf.batch, cf.V, cf.H, cf.W, cf.K, cf.scale, p.P, cf.res_hidden,
                                       cf.dec_hidden, p.max_core_h, p.max_core_w, st);
    }
    if (cf.precision == ORBIT2_BF16 && c->tma_stitch &&
        launch_stitch_tma(reinterpret_cast<const __nv_bfloat16*>(tile_out_dev), (int64_t)cf.batch * cd.chunk_core,
                          input_dev, out_dev, cd, cmap, cf.batch, cf.V, cf.H, cf.W, cf.K, cf.scale, p.P, p.max_core_h,
                          p.max_core_w, st))
      return true;
    if (cf.precision == ORBIT2_BF16)
      launch_stitch<__nv_bfloat16>(reinterpret_cast<const __nv_bfloat16*>(tile_out_dev), input_dev, out_dev, cd, cmap,
                                   cf.batch, cf.V, cf.H, cf.W, cf.K, cf.scale, p.P, p.max_core_h, st);
    else
      launch_stitch<float>(reinterpret_cast<const float*>(tile_out_dev), input_dev, out_dev, cd, cmap, cf.batch, cf.V,
                           cf.H, cf.W, cf.K, cf.scale, p.P, p.max_core_h, st);
    return true;
  });
}

orbit2_status orbit2_stitch(void* ctx, const void* tile_out_dev, const float* input_dev, int32_t tile_begin,
                            int32_t tile_count, float* out_dev, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (!tile_out_dev || !input_dev || !out_dev || !aligned16(tile_out_dev) || !aligned16(input_dev) ||
      !aligned16(out_dev))
    return set_err(ORBIT2_E_INVALID, "tile_out_dev/input_dev/out_dev: null or not 16-byte aligned");
  ORBIT2_TRY(check_range(c, tile_begin, tile_count));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Plan& p = c->plan;
  const orbit2_config& cf = p.cfg;
  const ChunkDev cd = chunk_dev(c, make_chunk(p, tile_begin, tile_count));
  const int32_t* cmap = c->at<int32_t>(p.lay.cmap);
  return run(c, "stitch_residual", st, [&] {
    if (cf.res_hidden || cf.dec_hidden) {   // residual (R31) / decoder (R32) convolutions
      const float* wr = c->at<float>(p.lay.rconv);
      const float* wd = c->at<float>(p.lay.dconv);
      if (cf.precision == ORBIT2_BF16)
        return launch_stitch_conv<__nv_bfloat16>(reinterpret_cast<const __nv_bfloat16*>(tile_out_dev), input_dev,
                                                 out_dev, cd, cmap, wr, wd, cf.batch, cf.V, cf.H, cf.W, cf.K, cf.scale,
                                                 p.P, cf.res_hidden, cf.dec_hidden, p.max_core_h, p.max_core_w, st);
      return launch_stitch_conv<float>(reinterpret_cast<const float*>(tile_out_dev), input_dev, out_dev, cd, cmap, wr,
                                       wd, cf.batch, cf.V, cf.H, cf.W, cf.K, cf.scale, p.P, cf.res_hidden,
                                       cf.dec_hidden, p.max_core_h, p.max_core_w, st);
    }
    if (cf.precision == ORBIT2_BF16 && c->tma_stitch &&
        launch_stitch_tma(reinterpret_cast<const __nv_bfloat16*>(tile_out_dev), (int64_t)cf.batch * cd.chunk_core,
                          input_dev, out_dev, cd, cmap, cf.batch, cf.V, cf.H, cf.W, cf.K, cf.scale, p.P, p.max_core_h,
                          p.max_core_w, st))
      return true;
    if (cf.precision == ORBIT2_BF16)
      launch_stitch<__nv_bfloat16>(reinterpret_cast<const __nv_bfloat16*>(tile_out_dev), input_dev, out_dev, cd,
                                   cmap, cf.batch, cf.V, cf.H, cf.W, cf.K, cf.scale, p.P, p.max_core_h, st);
    else
      launch_stitch<float>(reinterpret_cast<const float*>(tile_out_dev), input_dev, out_dev, cd, cmap, cf.batch,
                           cf.V, cf.H, cf.W, cf.K, cf.scale, p.P, p.max_core_h, st);
    return true;
  });
}

// ---------------------------------------------------------------------------
// Peer-memory TILES sequence parallelism (include/orbit2.h, orbit2_comm_*)
// ---------------------------------------------------------------------------
orbit2_status orbit2_ipc_export(const void* dev_ptr, orbit2_ipc_handle* out) {
  if (!dev_ptr || !out) return set_err(ORBIT2_E_INVALID, "dev_ptr/out: null");
  void* base = nullptr;
  size_t bytes = 0;
  if (!alloc_range(dev_ptr, &base, &bytes))
    return set_err(ORBIT2_E_CUDA, "orbit2_ipc_export: cuMemGetAddressRange failed (not a device allocation?)");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, base);
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
  static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t size");
  std::memcpy(out->handle, &h, 64);
  out->offset = reinterpret_cast<const uint8_t*>(dev_ptr) - reinterpret_cast<const uint8_t*>(base);
  out->bytes = (int64_t)bytes;
  return ORBIT2_OK;
}

namespace {
// Open a peer allocation once per distinct handle (two buffers of a peer may share
// one allocation of its caching allocator) and return the mapped buffer pointer.
orbit2_status open_peer(Ctx* c, std::vector<std::pair<orbit2_ipc_handle, void*>>* seen, const orbit2_ipc_handle& h,
                        int64_t need, void** out) {
  if (h.offset < 0 || need < 0 || h.offset + need > h.bytes)
    return set_err(ORBIT2_E_INVALID, "orbit2_comm_init: a peer buffer is smaller than the plan needs");
  void* base = nullptr;
  for (auto& s : *seen)
    if (std::memcmp(s.first.handle, h.handle, 64) == 0) base = s.second;
  if (!base) {
    cudaIpcMemHandle_t ih;
    std::memcpy(&ih, h.handle, 64);
    cudaError_t e = cudaIpcOpenMemHandle(&base, ih, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess)
      return set_err(ORBIT2_E_CUDA, std::string("cudaIpcOpenMemHandle (peer-to-peer over NVLink): ") +
                                        cudaGetErrorString(e));
    c->opened.push_back(base);
    seen->push_back({h, base});
  }
  *out = reinterpret_cast<uint8_t*>(base) + h.offset;
  return ORBIT2_OK;
}
}  // namespace

orbit2_status orbit2_comm_init(void* ctx, int32_t gather_root, float* input_dev, float* out_dev,
                               const orbit2_ipc_handle* ws_h, const orbit2_ipc_handle* in_h,
                               const orbit2_ipc_handle* out_h) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (c->comm) return set_err(ORBIT2_E_STATE, "orbit2_comm_init: already initialised");
  const Plan& p = c->plan;
  const orbit2_config& cf = p.cfg;
  const int R = cf.world_size, me = cf.rank;
  if (!ws_h || !in_h) return set_err(ORBIT2_E_INVALID, "workspace_handles/input_handles: null");
  if (!input_dev || !aligned16(input_dev)) return set_err(ORBIT2_E_INVALID, "input_dev: null or not 16-byte aligned");
  if (gather_root < -1 || gather_root >= R) return set_err(ORBIT2_E_INVALID, "gather_root: outside [-1, world_size)");
  const bool own_out = gather_root < 0 || gather_root == me;
  if (own_out && (!out_dev || !aligned16(out_dev)))
    return set_err(ORBIT2_E_INVALID, "out_dev: null or not 16-byte aligned on the gather root / sharded output");
  if (gather_root >= 0 && gather_root != me && !out_h)
    return set_err(ORBIT2_E_INVALID, "out_handles: null with gather_root >= 0");
  const int64_t in_bytes = (int64_t)cf.batch * cf.V * cf.H * cf.W * 4;
  std::vector<std::pair<orbit2_ipc_handle, void*>> seen;
  std::vector<uint64_t*> sig(R, nullptr);
  std::vector<float*> inputs(R, nullptr);
  for (int r = 0; r < R; ++r) {
    if (r == me) {
      sig[r] = c->at<uint64_t>(p.lay.sig);
      inputs[r] = input_dev;
      continue;
    }
    void* w = nullptr;
    ORBIT2_TRY(open_peer(c, &seen, ws_h[r], p.lay.sig + 2LL * R * 8 + 64, &w));
    sig[r] = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(w) + p.lay.sig);
    void* x = nullptr;
    ORBIT2_TRY(open_peer(c, &seen, in_h[r], in_bytes, &x));
    inputs[r] = reinterpret_cast<float*>(x);
  }
  float* target = out_dev;
  if (!own_out) {
    void* o = nullptr;
    ORBIT2_TRY(open_peer(c, &seen, out_h[gather_root], p.info.out_bytes, &o));
    target = reinterpret_cast<float*>(o);
  }
  // push table: this rank's HALO SEND rectangles of every peer, with the peer's field
  std::vector<DevPush> push;
  for (int peer = 0; peer < R; ++peer) {
    if (peer == me) continue;
    const XferList& xl = p.xfer[((size_t)ORBIT2_XFER_HALO * R + peer) * 2 + ORBIT2_SEND];
    for (int i = 0; i < xl.count; ++i) {
      const DevRect& d = p.rects[(size_t)xl.start + i];
      push.push_back(DevPush{d.y0, d.y1, d.x0, d.x1, inputs[peer], 0});
    }
  }
  cudaError_t e = cudaSuccess;
  if (!push.empty())
    e = cudaMemcpy(c->at<void>(p.lay.push), push.data(), push.size() * sizeof(DevPush), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(c->at<void>(p.lay.sigtab), sig.data(), R * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemset(c->at<void>(p.lay.sig), 0, 2ULL * R * 8 + 64);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("orbit2_comm_init: ") + cudaGetErrorString(e));
  c->gather_root = gather_root;
  c->own_input = input_dev;
  c->target = target;
  c->epoch[0] = c->epoch[1] = 0;
  c->comm = true;
  return ORBIT2_OK;
}

orbit2_status orbit2_comm_target(void* ctx, float** out_dev) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !out_dev) return set_err(ORBIT2_E_INVALID, "ctx/out_dev: null");
  if (!c->comm) return set_err(ORBIT2_E_STATE, "orbit2_comm_target: orbit2_comm_init not called");
  *out_dev = c->target;
  return ORBIT2_OK;
}

static orbit2_status comm_barrier(Ctx* c, int slot, cudaStream_t st) {
  const Plan& p = c->plan;
  const uint64_t ep = ++c->epoch[slot];
  return run(c, "comm_barrier", st, [&] {
    launch_barrier(c->at<uint64_t*>(p.lay.sigtab), p.cfg.world_size, p.cfg.rank, slot, ep,
                   reinterpret_cast<uint32_t*>(c->at<uint8_t>(p.lay.sig) + 2LL * p.cfg.world_size * 8), st);
    return true;
  });
}

orbit2_status orbit2_halo_exchange(void* ctx, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (!c->comm) return set_err(ORBIT2_E_STATE, "orbit2_halo_exchange: orbit2_comm_init not called");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Plan& p = c->plan;
  const orbit2_config& cf = p.cfg;
  if (p.n_push > 0)
    ORBIT2_TRY(run(c, "halo_push", st, [&] {
      launch_push(c->at<DevPush>(p.lay.push), p.n_push, cf.batch, cf.V, cf.H, cf.W, c->own_input, st);
      return true;
    }));
  return comm_barrier(c, 0, st);
}

orbit2_status orbit2_comm_barrier(void* ctx, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (!c->comm) return set_err(ORBIT2_E_STATE, "orbit2_comm_barrier: orbit2_comm_init not called");
  return comm_barrier(c, 1, reinterpret_cast<cudaStream_t>(stream));
}

orbit2_status orbit2_comm_status(void* ctx) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (!c->comm) return set_err(ORBIT2_E_STATE, "orbit2_comm_status: orbit2_comm_init not called");
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("orbit2_comm_status: ") + cudaGetErrorString(e));
  uint32_t err = 0;
  e = cudaMemcpy(&err, c->at<uint8_t>(c->plan.lay.sig) + 2LL * c->plan.cfg.world_size * 8, 4, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("orbit2_comm_status: ") + cudaGetErrorString(e));
  if (err != 0)
    return set_err(ORBIT2_E_STATE, "orbit2 comm barrier timed out (30 s) waiting for rank " + std::to_string(err - 1));
  return ORBIT2_OK;
}


/* ------------------------------------------------------------------------------
 * Training step (oracle/train.py T1-T4, readings R34-R36)
 * ---------------------------------------------------------------------------- */
static orbit2_status train_scope(const Ctx* c) {
  const Plan& p = c->plan;
  const orbit2_config& cf = p.cfg;
  if (cf.precision != ORBIT2_BF16) return set_err(ORBIT2_E_UNSUPPORTED, "training: BF16 precision only");
  if (p.d != 64) return set_err(ORBIT2_E_UNSUPPORTED, "training: head_dim 64 only (attention backward kernel)");
  if (cf.var_agg || cf.res_hidden || cf.dec_hidden)
    return set_err(ORBIT2_E_UNSUPPORTED, "training: var_agg / res_hidden / dec_hidden stages are out of scope (R36)");
  if (p.info.chunk_tiles < p.info.n_local_tiles)
    return set_err(ORBIT2_E_UNSUPPORTED, "training: one call over every rank-local tile (chunk_tiles = 0)");
  if (p.D > 1024 || p.D % 128)
    return set_err(ORBIT2_E_UNSUPPORTED, "training: embed a multiple of 128 up to 1024 (LayerNorm backward kernel)");
  return ORBIT2_OK;
}

static TrainLay train_layout(const Plan& p) {
  TrainLay t;
  const int64_t D = p.D, L = p.cfg.depth, H = p.cfg.heads;
  t.rows = p.lay.mrow;
  t.rows_core = p.lay.mcore;
  t.nh_pad = round_up(p.Nh, 64);
  int64_t off = 0;
  auto take = [&](int64_t bytes) { int64_t o = off; off = round_up(off + bytes, 1024); return o; };
  const int64_t R = t.rows, RC = t.rows_core;
  for (int64_t l = 0; l < L; ++l) {
    t.zin.push_back(take(R * D * 4));
    t.xn1.push_back(take(R * D * 2));
    t.qkv.push_back(take(R * 3 * D * 2));
    t.ao.push_back(take(R * D * 2));
    t.lse.push_back(take(H * R * 4));
    t.zmid.push_back(take(R * D * 4));
    t.xn2.push_back(take(R * D * 2));
    t.gdash.push_back(take(R * 4 * D * 2));
    t.hact.push_back(take(R * 4 * D * 2));
  }
  t.zfin = take(R * D * 4);
  t.hin = take(RC * D * 2);
  t.dz = take(R * D * 4);
  t.dz_bf = take(R * D * 2);
  t.dzm = take(R * D * 4);
  t.dzm_bf = take(R * D * 2);
  t.dh = take(R * 4 * D * 2);
  t.dxn = take(R * D * 4);
  t.dao = take(R * D * 2);
  t.delta = take(H * R * 4);
  t.dq = take(R * D * 4);
  t.dqkv = take(R * 3 * D * 2);
  t.dg = take(RC * t.nh_pad * 2);
  t.dhin = take(RC * D * 4);
  t.latw = take((int64_t)p.cfg.scale * p.cfg.H * 4);
  t.zero = take(4 * D * 4 + t.nh_pad * 4);
  for (int64_t l = 0; l < L; ++l) {
    t.wqkv_t.push_back(take(D * 3 * D * 2));
    t.wo_t.push_back(take(D * D * 2));
    t.w1_t.push_back(take(D * 4 * D * 2));
    t.w2_t.push_back(take(4 * D * D * 2));
  }
  t.wh_t = take(D * t.nh_pad * 2);
  t.total = off;
  return t;
}

orbit2_status orbit2_train_plan(void* ctx, orbit2_train_info* info) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c || !info) return set_err(ORBIT2_E_INVALID, "ctx/info: null");
  ORBIT2_TRY(train_scope(c));
  const Plan& p = c->plan;
  const TrainLay t = train_layout(p);
  info->workspace_bytes = t.total;
  info->canonical_weight_count = c->wl.c_total;
  // algorithmic FLOPs per sample: forward (every query of every block) + backward
  // (input and weight gradients of every GEMM except the patches' input gradient;
  // attention: S recomputed, dP, dV, dK, dQ = 2.5x its forward)
  const double D = p.D, L = p.cfg.depth, Din = p.Din, Nh = p.Nh;
  const double n = (double)p.info.local_tokens, nc = (double)p.info.local_core_tokens;
  double n2 = 0.0;
  for (int32_t i = 0; i < p.info.n_local_tiles; ++i) n2 += (double)p.dev[i].n_tokens * p.dev[i].n_tokens;
  const double gemm = L * 24.0 * D * D * n + 2.0 * Din * D * n + 2.0 * D * Nh * nc;
  const double attn = L * 4.0 * D * n2;
  info->fwd_flops_per_sample = gemm + attn;
  info->flops_per_sample = (gemm + attn) + (2.0 * gemm - 2.0 * Din * D * n) + 2.5 * attn;
  info->attn_bwd_flops_per_sample = 2.5 * attn;
  return ORBIT2_OK;
}

orbit2_status orbit2_train_bind(void* ctx, void* train_ws_dev, size_t bytes, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  ORBIT2_TRY(train_scope(c));
  if (!train_ws_dev || !aligned16(train_ws_dev)) return set_err(ORBIT2_E_INVALID, "train_ws_dev: null or unaligned");
  TrainLay t = train_layout(c->plan);
  if ((int64_t)bytes < t.total)
    return set_err(ORBIT2_E_INVALID, "train workspace: " + std::to_string(bytes) + " bytes < " +
                                         std::to_string(t.total) + " (orbit2_train_plan)");
  c->tl = t;
  c->tws = reinterpret_cast<uint8_t*>(train_ws_dev);
  c->train_prepared = false;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // rows past M of every buffer stay zero (TMA tiles read up to the 128-row padding)
  cudaError_t e = cudaMemsetAsync(c->tws, 0, (size_t)t.total, st);
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("train_bind memset: ") + cudaGetErrorString(e));
  const int sH = c->plan.cfg.scale * c->plan.cfg.H;
  return run(c, "lat_weights", st, [&] {
    launch_lat_weights(c->tat<float>(t.latw), sH, st);
    return true;
  });
}

orbit2_status orbit2_train_prepare(void* ctx, const float* canonical_dev, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (!c->tws) return set_err(ORBIT2_E_STATE, "orbit2_train_prepare: orbit2_train_bind not called");
  if (!canonical_dev) return set_err(ORBIT2_E_INVALID, "canonical_dev: null");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Plan& p = c->plan;
  const WeightLayout& w = c->wl;
  const TrainLay& t = c->tl;
  const int D = p.D;
  typedef __nv_bfloat16 bf16;
  ORBIT2_TRY(run(c, "weight_transpose", st, [&] {
    for (int l = 0; l < p.cfg.depth; ++l) {
      const LayerW& L = w.c_layers[l];
      launch_transpose_bf16(canonical_dev + L.w_qkv, 3 * D, D, c->tat<bf16>(t.wqkv_t[l]), 3 * D, st);
      launch_transpose_bf16(canonical_dev + L.w_o, D, D, c->tat<bf16>(t.wo_t[l]), D, st);
      launch_transpose_bf16(canonical_dev + L.w_1, 4 * D, D, c->tat<bf16>(t.w1_t[l]), 4 * D, st);
      launch_transpose_bf16(canonical_dev + L.w_2, D, 4 * D, c->tat<bf16>(t.w2_t[l]), D, st);
    }
    launch_transpose_bf16(canonical_dev + w.c_w_h, p.Nh, D, c->tat<bf16>(t.wh_t), t.nh_pad, st);
    return true;
  }));
  c->train_prepared = true;
  return ORBIT2_OK;
}

orbit2_status orbit2_train_forward(void* ctx, const void* packed_w, const float* input_dev, void* tile_out_dev,
                                   void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (!c->tws) return set_err(ORBIT2_E_STATE, "orbit2_train_forward: orbit2_train_bind not called");
  if (!packed_w || !input_dev || !tile_out_dev || !aligned16(packed_w) || !aligned16(input_dev) ||
      !aligned16(tile_out_dev))
    return set_err(ORBIT2_E_INVALID, "packed_w/input_dev/tile_out_dev: null or not 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Plan& p = c->plan;
  const orbit2_config& cf = p.cfg;
  const Layout& ly = p.lay;
  const WeightLayout& w = c->wl;
  const TrainLay& t = c->tl;
  typedef __nv_bfloat16 bf16;
  const uint8_t* W8 = reinterpret_cast<const uint8_t*>(packed_w);
  auto wf = [&](int64_t off) { return reinterpret_cast<const float*>(W8 + off); };
  const Chunk ch = make_chunk(p, 0, p.info.n_local_tiles);
  const ChunkDev cd = chunk_dev(c, ch);
  const int B = cf.batch;
  const int64_t M = (int64_t)B * ch.chunk_tokens, Mc = (int64_t)B * ch.chunk_core;
  const int64_t D = p.D, F = 4LL * p.D, R = t.rows;
  int2* rowinfo = c->at<int2>(ly.rowinfo);
  bf16* patches = c->at<bf16>(ly.patches);
  auto gemm = [&](const char* name, int epi, int out_bf, const void* A, int64_t lda, int64_t wo, int64_t n,
                  int64_t k, int64_t rows, EpiParams ep, int64_t acols = 0) {
    GemmOperand a{A, R, lda, acols}, b{W8 + wo, n, k};
    ep.M = (int32_t)rows;
    ep.N = (int32_t)n;
    return run(c, name, st, [&] {
      ep.single_cta = c->single_cta_gemm;
      return launch_gemm_tc(epi, out_bf, a, b, rows, n, k, ep, st);
    });
  };
  int64_t lda_patch = ly.din_pad, cols_patch = 0;
  if (cf.halo_mode == ORBIT2_HALO_CLAMP && !c->simt_gather) {
    bool ok = false;
    ORBIT2_TRY(run(c, "tile_gather", st, [&] {
      ok = launch_gather_tma(input_dev, patches, rowinfo, cd, B, cf.V, cf.H, cf.W, cf.patch, p.Din, ly.ld_patch,
                             p.max_pad_h, p.max_pad_w, st);
      return true;
    }));
    if (ok) {
      lda_patch = ly.ld_patch;
      cols_patch = p.Din;
    }
  }
  if (cols_patch == 0)
    ORBIT2_TRY(run(c, "tile_gather", st, [&] {
      launch_gather<bf16>(input_dev, patches, rowinfo, cd, B, cf.V, cf.H, cf.W, cf.patch, p.Din, ly.din_pad,
                          p.max_pad_h, st);
      return true;
    }));
  c->tl_lda_patch = lda_patch;
  c->tl_cols_patch = cols_patch ? cols_patch : p.Din;
  EpiParams emb{};
  emb.bias = wf(w.bias_e); emb.ldc = D;
  emb.rowinfo = rowinfo; emb.pos_u = c->at<float>(ly.pos_u); emb.pos_w = c->at<float>(ly.pos_w);
  emb.pos_off = cf.halo; emb.half = (int32_t)(D / 2);
  emb.C = cf.depth > 0 ? c->tat<float>(t.zin[0]) : c->tat<float>(t.zfin);
  {
    GemmOperand a{patches, ly.mrow, lda_patch, cols_patch}, b{W8 + w.w_e, D, ly.din_pad};
    emb.M = (int32_t)M;
    emb.N = (int32_t)D;
    ORBIT2_TRY(run(c, "embed_gemm", st, [&] {
      emb.single_cta = c->single_cta_gemm;
      return launch_gemm_tc(EPI_EMBED, 0, a, b, M, D, ly.din_pad, emb, st);
    }));
  }
  for (int l = 0; l < cf.depth; ++l) {
    const LayerW& L = w.layers[l];
    float* zin = c->tat<float>(t.zin[l]);
    float* zmid = c->tat<float>(t.zmid[l]);
    float* zout = l + 1 < cf.depth ? c->tat<float>(t.zin[l + 1]) : c->tat<float>(t.zfin);
    bf16* xn1 = c->tat<bf16>(t.xn1[l]);
    bf16* qkv = c->tat<bf16>(t.qkv[l]);
    bf16* ao = c->tat<bf16>(t.ao[l]);
    bf16* xn2 = c->tat<bf16>(t.xn2[l]);
    ORBIT2_TRY(run(c, "layernorm", st, [&] {
      launch_layernorm<bf16>(zin, wf(L.ln1_g), wf(L.ln1_b), xn1, M, (int)D, nullptr, st);
      return true;
    }));
    EpiParams e{};
    e.bias = wf(L.b_qkv); e.C = qkv; e.ldc = 3 * D;
    ORBIT2_TRY(gemm("qkv_gemm", EPI_BIAS, 1, xn1, D, L.w_qkv, 3 * D, D, M, e));
    ORBIT2_TRY(run(c, "tile_attention", st, [&] {
      return launch_attention_tc(qkv, R, ao, cd, B, (int)D, cf.heads, p.d, st, c->tat<float>(t.lse[l]), R);
    }));
    e = EpiParams{}; e.bias = wf(L.b_o); e.C = zmid; e.ldc = D; e.aux = zin;
    ORBIT2_TRY(gemm("oproj_gemm", EPI_RESID, 0, ao, D, L.w_o, D, D, M, e));
    ORBIT2_TRY(run(c, "layernorm", st, [&] {
      launch_layernorm<bf16>(zmid, wf(L.ln2_g), wf(L.ln2_b), xn2, M, (int)D, nullptr, st);
      return true;
    }));
    e = EpiParams{}; e.bias = wf(L.b_1); e.C = c->tat<bf16>(t.hact[l]); e.ldc = F; e.aux = c->tat<bf16>(t.gdash[l]);
    ORBIT2_TRY(gemm("mlp_up_gemm", EPI_GELU, 1, xn2, D, L.w_1, F, D, M, e));
    e = EpiParams{}; e.bias = wf(L.b_2); e.C = zout; e.ldc = D; e.aux = zmid;
    ORBIT2_TRY(gemm("mlp_down_gemm", EPI_RESID, 0, c->tat<bf16>(t.hact[l]), F, L.w_2, D, F, M, e));
  }
  bf16* hin = c->tat<bf16>(t.hin);
  ORBIT2_TRY(run(c, "layernorm", st, [&] {
    launch_layernorm<bf16>(c->tat<float>(t.zfin), wf(w.lnf_g), wf(w.lnf_b), hin, Mc, (int)D, &cd, st);
    return true;
  }));
  EpiParams e{};
  e.bias = wf(w.b_h); e.C = tile_out_dev; e.ldc = p.Nh; e.M = (int32_t)Mc; e.N = p.Nh;
  {
    GemmOperand a{hin, t.rows_core, D, 0}, b{W8 + w.w_h, p.Nh, D};
    ORBIT2_TRY(run(c, "head_gemm", st, [&] {
      e.single_cta = c->single_cta_gemm;
      return launch_gemm_tc(EPI_BIAS, 1, a, b, Mc, p.Nh, D, e, st);
    }));
  }
  return ORBIT2_OK;
}

orbit2_status orbit2_loss(void* ctx, const float* out_dev, const float* truth_dev, float lambda, float delta,
                          int32_t geo, double* loss_dev, float* dout_dev, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (!c->tws) return set_err(ORBIT2_E_STATE, "orbit2_loss: orbit2_train_bind not called");
  if (!out_dev || !truth_dev || !loss_dev || !dout_dev) return set_err(ORBIT2_E_INVALID, "loss: null pointer");
  if (!(delta > 0.f) || !(lambda >= 0.f)) return set_err(ORBIT2_E_INVALID, "loss: delta must be > 0, lambda >= 0");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const orbit2_config& cf = c->plan.cfg;
  const int sH = cf.scale * cf.H, sW = cf.scale * cf.W;
  cudaError_t e = cudaMemsetAsync(loss_dev, 0, sizeof(double) * cf.batch, st);
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("loss memset: ") + cudaGetErrorString(e));
  return run(c, "bayesian_loss", st, [&] {
    launch_loss(out_dev, truth_dev, cf.batch, cf.K, sH, sW, lambda, delta, geo ? 1 : 0, c->tat<float>(c->tl.latw),
                loss_dev, dout_dev, st);
    return true;
  });
}

orbit2_status orbit2_train_backward(void* ctx, const void* packed_w, const float* dout_dev, float* grad_dev,
                                    void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  if (!c->tws || !c->train_prepared)
    return set_err(ORBIT2_E_STATE, "orbit2_train_backward: orbit2_train_bind / orbit2_train_prepare not called");
  if (!packed_w || !dout_dev || !grad_dev || !aligned16(grad_dev))
    return set_err(ORBIT2_E_INVALID, "packed_w/dout_dev/grad_dev: null or not 16-byte aligned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Plan& p = c->plan;
  const orbit2_config& cf = p.cfg;
  const Layout& ly = p.lay;
  const WeightLayout& w = c->wl;
  const TrainLay& t = c->tl;
  typedef __nv_bfloat16 bf16;
  const uint8_t* W8 = reinterpret_cast<const uint8_t*>(packed_w);
  auto wf = [&](int64_t off) { return reinterpret_cast<const float*>(W8 + off); };
  const Chunk ch = make_chunk(p, 0, p.info.n_local_tiles);
  const ChunkDev cd = chunk_dev(c, ch);
  const int B = cf.batch;
  const int64_t M = (int64_t)B * ch.chunk_tokens, Mc = (int64_t)B * ch.chunk_core;
  const int D = p.D, F = 4 * p.D;
  const int64_t R = t.rows;
  const float* zero = c->tat<float>(t.zero);
  auto memset0 = [&](void* ptr, size_t bytes) {
    cudaError_t e = cudaMemsetAsync(ptr, 0, bytes, st);
    return e == cudaSuccess ? ORBIT2_OK : set_err(ORBIT2_E_CUDA, std::string("memset: ") + cudaGetErrorString(e));
  };
  // input-gradient GEMM: C[rows][n] = A[rows][k] W^T-operand[n][k] (the transposed weights)
  auto dx = [&](const char* name, int epi, int out_bf, const void* A, int64_t arows, int64_t lda, const void* Bt,
                int64_t n, int64_t k, int64_t rows, void* C, int64_t ldc, const void* aux, int64_t acols = 0) {
    GemmOperand a{A, arows, lda, acols}, b{Bt, n, k};
    EpiParams ep{};
    ep.M = (int32_t)rows; ep.N = (int32_t)n; ep.bias = zero; ep.C = C; ep.ldc = ldc; ep.aux = aux;
    return run(c, name, st, [&] {
      ep.single_cta = c->single_cta_gemm;
      return launch_gemm_tc(epi, out_bf, a, b, rows, n, k, ep, st);
    });
  };
  auto wg = [&](const char* name, const void* dY, int64_t ldy, const void* X, int64_t ldx, int64_t rows, int n,
                int kc, int64_t gw, int64_t gb) {
    GemmOperand a{dY, rows, ldy, 0}, x{X, rows, ldx, 0};
    return run(c, name, st, [&] {
      return launch_wgrad_tc(a, x, rows, n, kc, grad_dev + gw, kc, gb >= 0 ? grad_dev + gb : nullptr, st);
    });
  };
  ORBIT2_TRY(memset0(grad_dev, (size_t)w.c_total * 4));
  // O6 backwards, then the head (g = LN_f(z_core) W_h^T + b_h)
  bf16* dg = c->tat<bf16>(t.dg);
  ORBIT2_TRY(run(c, "stitch_bwd", st, [&] {
    launch_stitch_bwd(dout_dev, dg, t.nh_pad, cd, B, cf.K, p.P, cf.scale * cf.H, cf.scale * cf.W, st);
    return true;
  }));
  bf16* hin = c->tat<bf16>(t.hin);
  ORBIT2_TRY(wg("wgrad_head", dg, t.nh_pad, hin, D, Mc, p.Nh, D, w.c_w_h, w.c_b_h));
  float* dhin = c->tat<float>(t.dhin);
  ORBIT2_TRY(dx("dx_head", EPI_BIAS, 0, dg, t.rows_core, t.nh_pad, c->tat<bf16>(t.wh_t), D, t.nh_pad, Mc, dhin, D,
                nullptr));
  float* dz = c->tat<float>(t.dz);
  bf16* dz_bf = c->tat<bf16>(t.dz_bf);
  ORBIT2_TRY(memset0(dz, (size_t)R * D * 4));
  ORBIT2_TRY(memset0(dz_bf, (size_t)R * D * 2));
  ORBIT2_TRY(run(c, "ln_bwd", st, [&] {   // LN_f over the core rows (R16: halo rows get no gradient)
    return launch_ln_bwd(dhin, D, c->tat<float>(t.zfin), wf(w.lnf_g), nullptr, dz, dz_bf, Mc, D, cd.core_row + ch.core0,
                         ch.chunk_core, ch.chunk_tokens, ch.tok0, grad_dev + w.c_lnf_g, grad_dev + w.c_lnf_b, st);
  }));
  float* dzm = c->tat<float>(t.dzm);
  bf16* dzm_bf = c->tat<bf16>(t.dzm_bf);
  bf16* dh = c->tat<bf16>(t.dh);
  float* dxn = c->tat<float>(t.dxn);
  bf16* dao = c->tat<bf16>(t.dao);
  bf16* dqkv = c->tat<bf16>(t.dqkv);
  float* dq = c->tat<float>(t.dq);
  float* dlt = c->tat<float>(t.delta);
  for (int l = cf.depth - 1; l >= 0; --l) {
    const LayerW& CL = w.c_layers[l];
    const LayerW& L = w.layers[l];
    // z_out = zmid + GELU(h) W_2^T + b_2,  h = LN2(zmid) W_1^T + b_1
    ORBIT2_TRY(wg("wgrad_w2", dz_bf, D, c->tat<bf16>(t.hact[l]), F, M, D, F, CL.w_2, CL.b_2));
    ORBIT2_TRY(dx("dx_mlp_down", EPI_DGELU, 1, dz_bf, R, D, c->tat<bf16>(t.w2_t[l]), F, D, M, dh, F,
                  c->tat<bf16>(t.gdash[l])));
    ORBIT2_TRY(wg("wgrad_w1", dh, F, c->tat<bf16>(t.xn2[l]), D, M, F, D, CL.w_1, CL.b_1));
    ORBIT2_TRY(dx("dx_mlp_up", EPI_BIAS, 0, dh, R, F, c->tat<bf16>(t.w1_t[l]), D, F, M, dxn, D, nullptr));
    ORBIT2_TRY(run(c, "ln_bwd", st, [&] {
      return launch_ln_bwd(dxn, D, c->tat<float>(t.zmid[l]), wf(L.ln2_g), dz, dzm, dzm_bf, M, D, nullptr, 0, 0, 0,
                           grad_dev + CL.ln2_g, grad_dev + CL.ln2_b, st);
    }));
    // zmid = z_in + attn W_o^T + b_o
    bf16* ao = c->tat<bf16>(t.ao[l]);
    ORBIT2_TRY(wg("wgrad_wo", dzm_bf, D, ao, D, M, D, D, CL.w_o, CL.b_o));
    ORBIT2_TRY(dx("dx_oproj", EPI_BIAS, 1, dzm_bf, R, D, c->tat<bf16>(t.wo_t[l]), D, D, M, dao, D, nullptr));
    // attention (per tile, per head)
    ORBIT2_TRY(run(c, "attn_delta", st, [&] {
      launch_delta(dao, ao, dlt, M, D, cf.heads, R, st);
      return true;
    }));
    ORBIT2_TRY(memset0(dq, (size_t)M * D * 4));
    ORBIT2_TRY(run(c, "attn_bwd", st, [&] {
      return launch_attention_bwd_tc(c->tat<bf16>(t.qkv[l]), dao, R, c->tat<float>(t.lse[l]), dlt, R, dq, dqkv, cd, B,
                                     D, cf.heads, p.d, st);
    }));
    ORBIT2_TRY(run(c, "dq_convert", st, [&] {
      launch_dq_convert(dq, dqkv, M, D, st);
      return true;
    }));
    // qkv = LN1(z_in) W_qkv^T + b_qkv
    ORBIT2_TRY(wg("wgrad_wqkv", dqkv, 3 * D, c->tat<bf16>(t.xn1[l]), D, M, 3 * D, D, CL.w_qkv, CL.b_qkv));
    ORBIT2_TRY(dx("dx_qkv", EPI_BIAS, 0, dqkv, R, 3 * D, c->tat<bf16>(t.wqkv_t[l]), D, 3 * D, M, dxn, D, nullptr));
    ORBIT2_TRY(run(c, "ln_bwd", st, [&] {
      return launch_ln_bwd(dxn, D, c->tat<float>(t.zin[l]), wf(L.ln1_g), dzm, dz, dz_bf, M, D, nullptr, 0, 0, 0,
                           grad_dev + CL.ln1_g, grad_dev + CL.ln1_b, st);
    }));
  }
  // z0 = patches W_e^T + b_e + e_s + pi
  ORBIT2_TRY(wg("wgrad_embed", dz_bf, D, c->at<bf16>(ly.patches), c->tl_lda_patch, M, D, p.Din, w.c_w_e, w.c_b_e));
  cudaError_t e = cudaMemcpyAsync(grad_dev + w.c_e_s, grad_dev + w.c_b_e, (size_t)D * 4, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("grad e_s copy: ") + cudaGetErrorString(e));
  return ORBIT2_OK;
}


/* ------------------------------------------------------------------------------
 * Adaptive spatial compression (oracle/compress.py, R37-R40)
 * ---------------------------------------------------------------------------- */
struct CompressLay {
  int64_t tmp, tmp2, mag, dir, lab, gmax, changed, flag, bsum;
  int64_t rows, wext, proj;   // tokenize / detokenize (C, embed > 0)
  int64_t total;
  int levels;
};

static orbit2_status compress_check(const orbit2_compress_config* c, CompressLay* ly) {
  if (!c) return set_err(ORBIT2_E_INVALID, "compress cfg: null");
  if (c->batch < 1 || c->H < 3 || c->W < 3) return set_err(ORBIT2_E_INVALID, "compress: batch >= 1, H, W >= 3");
  if (c->min_side < 1 || c->max_side < 2 * c->min_side || c->max_side % c->min_side ||
      ((c->max_side / c->min_side) & (c->max_side / c->min_side - 1)) || c->max_side / c->min_side > 64)
    return set_err(ORBIT2_E_INVALID, "compress: max_side must be min_side * 2^k, 1 <= k <= 6");
  if (c->H % c->max_side || c->W % c->max_side)
    return set_err(ORBIT2_E_INVALID, "compress: H, W must be multiples of max_side (pad by edge replication)");
  float w[32];
  int r = 0;
  if (!compress_taps(c->sigma, w, &r)) return set_err(ORBIT2_E_INVALID, "compress: sigma must be in (0, 8/3]");
  if (!(c->low_frac > 0.f) || !(c->low_frac <= c->high_frac) || !std::isfinite(c->threshold))
    return set_err(ORBIT2_E_INVALID, "compress: 0 < low_frac <= high_frac, finite threshold");
  const int64_t n = (int64_t)c->batch * c->H * c->W;
  const int64_t cells = (int64_t)c->batch * (c->H / c->min_side) * (c->W / c->min_side);
  int64_t off = 0;
  auto take = [&](int64_t b) { int64_t o = off; off = round_up(off + b, 256); return o; };
  ly->tmp = take(n * 4);
  ly->tmp2 = take(n * 4);
  ly->mag = take(n * 4);
  ly->dir = take(n);
  ly->lab = take(n);
  ly->gmax = take((int64_t)c->batch * 4);
  ly->changed = take(4);
  ly->flag = take(cells * 4);
  ly->bsum = take(((cells + 1023) / 1024) * 4);
  ly->levels = 1;
  while ((c->min_side << (ly->levels - 1)) < c->max_side) ++ly->levels;
  const int64_t K = (int64_t)std::max(c->C, 0) * c->min_side * c->min_side;
  const int64_t D = std::max(c->embed, 0);
  ly->rows = take(cells * (K + ly->levels) * 4);
  ly->wext = take(D * (K + ly->levels) * 4);
  ly->proj = take(cells * K * 4);
  ly->total = off;
  return ORBIT2_OK;
}

orbit2_status orbit2_compress_plan(const orbit2_compress_config* cfg, int64_t* workspace_bytes, int64_t* max_patches) {
  CompressLay ly;
  ORBIT2_TRY(compress_check(cfg, &ly));
  if (workspace_bytes) *workspace_bytes = ly.total;
  if (max_patches) *max_patches = (int64_t)cfg->batch * (cfg->H / cfg->min_side) * (cfg->W / cfg->min_side);
  return ORBIT2_OK;
}

orbit2_status orbit2_compress_partition(const orbit2_compress_config* cfg, const float* image_dev, void* ws,
                                        size_t ws_bytes, uint8_t* edges_dev, int32_t* patches_dev,
                                        int32_t* offsets_dev, int32_t* n_host, void* stream) {
  CompressLay ly;
  ORBIT2_TRY(compress_check(cfg, &ly));
  if (!image_dev || !ws || !patches_dev || !offsets_dev) return set_err(ORBIT2_E_INVALID, "compress: null pointer");
  if ((int64_t)ws_bytes < ly.total) return set_err(ORBIT2_E_INVALID, "compress: workspace smaller than planned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* w8 = reinterpret_cast<uint8_t*>(ws);
  const int B = cfg->batch, H = cfg->H, W = cfg->W;
  int passes = 0;
  launch_canny(image_dev, reinterpret_cast<float*>(w8 + ly.tmp), reinterpret_cast<float*>(w8 + ly.tmp2),
               reinterpret_cast<float*>(w8 + ly.mag), w8 + ly.dir, w8 + ly.lab,
               reinterpret_cast<unsigned*>(w8 + ly.gmax), reinterpret_cast<int*>(w8 + ly.changed), B, H, W,
               cfg->sigma, cfg->low_frac, cfg->high_frac, st, &passes);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("compress canny: ") + cudaGetErrorString(e));
  if (edges_dev) launch_edges(w8 + ly.lab, edges_dev, (int64_t)B * H * W, st);
  launch_quadtree(w8 + ly.lab, reinterpret_cast<int32_t*>(w8 + ly.flag), reinterpret_cast<int32_t*>(w8 + ly.bsum),
                  offsets_dev + B, patches_dev, offsets_dev, B, H, W, cfg->min_side, cfg->max_side,
                  (double)cfg->threshold, st);
  e = cudaGetLastError();
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("compress quadtree: ") + cudaGetErrorString(e));
  if (n_host) {
    e = cudaMemcpyAsync(n_host, offsets_dev + B, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("compress count: ") + cudaGetErrorString(e));
  }
  return ORBIT2_OK;
}

orbit2_status orbit2_compress_tokenize(const orbit2_compress_config* cfg, void* ws, size_t ws_bytes,
                                       const float* feat_dev, const int32_t* patches_dev, int32_t n,
                                       const float* w_tok, const float* b_tok, const float* e_scale,
                                       float* tokens_dev, void* stream) {
  CompressLay ly;
  ORBIT2_TRY(compress_check(cfg, &ly));
  if (cfg->C < 1 || cfg->embed < 1) return set_err(ORBIT2_E_INVALID, "compress tokenize: C, embed >= 1");
  if (!ws || (int64_t)ws_bytes < ly.total) return set_err(ORBIT2_E_INVALID, "compress tokenize: workspace");
  if (n < 0 || !w_tok || !e_scale || (n > 0 && (!feat_dev || !patches_dev || !b_tok || !tokens_dev)))
    return set_err(ORBIT2_E_INVALID, "compress tokenize: null pointer or n < 0");
  if (n > (int64_t)cfg->batch * (cfg->H / cfg->min_side) * (cfg->W / cfg->min_side))
    return set_err(ORBIT2_E_INVALID, "compress tokenize: n exceeds the leaf capacity");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* w8 = reinterpret_cast<uint8_t*>(ws);
  launch_tokenize(feat_dev, patches_dev, n, cfg->C, cfg->H, cfg->W, cfg->min_side, cfg->embed, ly.levels, w_tok, b_tok,
                  e_scale, reinterpret_cast<float*>(w8 + ly.rows), reinterpret_cast<float*>(w8 + ly.wext), tokens_dev,
                  st);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ORBIT2_OK : set_err(ORBIT2_E_CUDA, std::string("compress tokenize: ") + cudaGetErrorString(e));
}

orbit2_status orbit2_compress_detokenize(const orbit2_compress_config* cfg, void* ws, size_t ws_bytes,
                                         const float* tokens_dev, const int32_t* patches_dev, int32_t n,
                                         const float* w_dec, const float* b_dec, const float* w_sm, const float* b_sm,
                                         float* work_dev, float* out_dev, void* stream) {
  CompressLay ly;
  ORBIT2_TRY(compress_check(cfg, &ly));
  if (cfg->C < 1 || cfg->embed < 1) return set_err(ORBIT2_E_INVALID, "compress detokenize: C, embed >= 1");
  if (!ws || (int64_t)ws_bytes < ly.total) return set_err(ORBIT2_E_INVALID, "compress detokenize: workspace");
  if (n < 0 || !w_sm || !b_sm || !work_dev || !out_dev || (n > 0 && (!tokens_dev || !patches_dev || !w_dec || !b_dec)))
    return set_err(ORBIT2_E_INVALID, "compress detokenize: null pointer or n < 0");
  if (n > (int64_t)cfg->batch * (cfg->H / cfg->min_side) * (cfg->W / cfg->min_side))
    return set_err(ORBIT2_E_INVALID, "compress detokenize: n exceeds the leaf capacity");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* w8 = reinterpret_cast<uint8_t*>(ws);
  launch_detokenize(tokens_dev, patches_dev, n, cfg->batch, cfg->C, cfg->H, cfg->W, cfg->min_side, cfg->embed, w_dec,
                    b_dec, w_sm, b_sm, reinterpret_cast<float*>(w8 + ly.proj), work_dev, out_dev, st);
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ORBIT2_OK
                          : set_err(ORBIT2_E_CUDA, std::string("compress detokenize: ") + cudaGetErrorString(e));
}

/* ------------------------------------------------------------------------------
 * The Reslim forward on compressed tokens (R41; oracle/compress.py K5)
 * ---------------------------------------------------------------------------- */
struct CfwdLay {
  int64_t field, cws_part, leaves, offsets, ext, tok, g, tiles, qblk, qpair, qpc, qg3, qg3c, core_row, total;
  int64_t part_bytes, cap, tabcap;
  int Hq, Wq, T, imgs;
};

static orbit2_status cfwd_layout(const Ctx* c, const orbit2_compression* cp, CfwdLay* L,
                                 orbit2_compress_config* cc) {
  const Plan& p = c->plan;
  const orbit2_config& cf = p.cfg;
  if (!cp) return set_err(ORBIT2_E_INVALID, "compression: null");
  if (cf.precision != ORBIT2_BF16 || cf.var_agg || cf.dec_hidden || cf.res_hidden)
    return set_err(ORBIT2_E_UNSUPPORTED, "compressed forward: a BF16 context without var_agg / dec_hidden / "
                                         "res_hidden (R41, R42)");
  if (p.info.chunk_tiles < p.info.n_local_tiles)
    return set_err(ORBIT2_E_UNSUPPORTED, "compressed forward: one call over every rank-local tile (chunk_tiles = 0)");
  const int mx = cp->max_side;
  L->T = p.info.n_local_tiles;
  L->imgs = cf.batch * L->T;
  L->Hq = (int)round_up(p.max_pad_h, mx);   // R42: every tile's field padded to one shape
  L->Wq = (int)round_up(p.max_pad_w, mx);
  *cc = orbit2_compress_config{L->imgs, L->Hq, L->Wq, 1, 1, mx, p.D, cp->threshold, cp->sigma, cp->low_frac,
                               cp->high_frac};
  int64_t ws = 0, maxp = 0;
  ORBIT2_TRY(orbit2_compress_plan(cc, &ws, &maxp));
  const int64_t I = L->imgs;
  L->cap = maxp;                                         // leaves (upper bound)
  L->tabcap = L->cap / 128 + 2 * I + 2;                  // 128-token blocks of all images
  int64_t off = 0;
  auto take = [&](int64_t b) { int64_t o = off; off = round_up(off + b, 256); return o; };
  L->field = take(I * L->Hq * L->Wq * 4);
  L->part_bytes = ws;
  L->cws_part = take(ws);
  L->leaves = take(L->cap * 16);
  L->offsets = take((I + 1) * 4);
  L->ext = take(I * 8);
  L->tok = take(L->cap * p.D * 4);
  L->g = take(L->cap * round_up(p.Nh, 8) * 2);
  L->tiles = take((I + 1) * (int64_t)sizeof(DevTile));
  L->qblk = take(L->tabcap * 4);
  L->qpair = take(L->tabcap * 4);
  L->qpc = take(L->tabcap * 4);
  L->qg3 = take(L->tabcap * 4);
  L->qg3c = take(L->tabcap * 4);
  L->core_row = take(4);
  L->total = off;
  return ORBIT2_OK;
}

orbit2_status orbit2_compressed_plan(void* ctx, const orbit2_compression* cp, int64_t* workspace_bytes,
                                     int32_t* levels) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  CfwdLay L;
  orbit2_compress_config cc;
  ORBIT2_TRY(cfwd_layout(c, cp, &L, &cc));
  if (workspace_bytes) *workspace_bytes = L.total;
  if (levels) {
    int l = 1;
    while ((1 << (l - 1)) < cp->max_side) ++l;
    *levels = l;
  }
  return ORBIT2_OK;
}

orbit2_status orbit2_compressed_forward(void* ctx, const void* packed_w, const float* input_dev,
                                        const orbit2_compression* cp, const float* e_scale_dev, void* cws,
                                        size_t cws_bytes, void* tile_out_dev, int32_t* leaves_dev,
                                        int32_t* n_tokens_host, void* stream) {
  Ctx* c = reinterpret_cast<Ctx*>(ctx);
  if (!c) return set_err(ORBIT2_E_INVALID, "ctx: null");
  CfwdLay L;
  orbit2_compress_config cc;
  ORBIT2_TRY(cfwd_layout(c, cp, &L, &cc));
  if (!packed_w || !input_dev || !e_scale_dev || !cws || !tile_out_dev || !aligned16(cws) || !aligned16(tile_out_dev))
    return set_err(ORBIT2_E_INVALID, "compressed forward: null or unaligned pointer");
  if ((int64_t)cws_bytes < L.total) return set_err(ORBIT2_E_INVALID, "compressed forward: workspace < planned");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const Plan& p = c->plan;
  const orbit2_config& cf = p.cfg;
  const Layout& ly = p.lay;
  const WeightLayout& w = c->wl;
  typedef __nv_bfloat16 bf16;
  const uint8_t* W8 = reinterpret_cast<const uint8_t*>(packed_w);
  auto wf = [&](int64_t off) { return reinterpret_cast<const float*>(W8 + off); };
  uint8_t* cw = reinterpret_cast<uint8_t*>(cws);
  const int B = cf.batch, T = L.T, I = L.imgs;
  const int64_t D = p.D, F = 4LL * p.D, mrow = ly.mrow;
  // 1-2: gather + patch embedding (O2, O3) of every padded-rectangle patch: z0 = the ctx's z
  const Chunk ch = make_chunk(p, 0, T);
  const ChunkDev cd = chunk_dev(c, ch);
  const int64_t M0 = (int64_t)B * ch.chunk_tokens;
  int2* rowinfo = c->at<int2>(ly.rowinfo);
  float* z = c->at<float>(ly.z);
  bf16* patches = c->at<bf16>(ly.patches);
  ORBIT2_TRY(run(c, "tile_gather", st, [&] {
    launch_gather<bf16>(input_dev, patches, rowinfo, cd, B, cf.V, cf.H, cf.W, cf.patch, p.Din, ly.din_pad,
                        p.max_pad_h, st);
    return true;
  }));
  {
    EpiParams emb{};
    emb.M = (int32_t)M0; emb.N = (int32_t)D; emb.bias = wf(w.bias_e); emb.C = z; emb.ldc = D;
    emb.rowinfo = rowinfo; emb.pos_u = c->at<float>(ly.pos_u); emb.pos_w = c->at<float>(ly.pos_w);
    emb.pos_off = cf.halo; emb.half = (int32_t)(D / 2);
    GemmOperand a{patches, mrow, ly.din_pad, 0}, b{W8 + w.w_e, D, ly.din_pad};
    ORBIT2_TRY(run(c, "embed_gemm", st, [&] {
      emb.single_cta = c->single_cta_gemm;
      return launch_gemm_tc(EPI_EMBED, 0, a, b, M0, D, ly.din_pad, emb, st);
    }));
  }
  // 3: every (sample, tile) rectangle's field and its partition (Canny + quad-tree, patch grid)
  float* field = reinterpret_cast<float*>(cw + L.field);
  ORBIT2_TRY(run(c, "compress_field", st, [&] {
    launch_cfield(z, cd, T, B, (int)D, L.Hq, L.Wq, field, st);
    return true;
  }));
  int32_t* leaves = reinterpret_cast<int32_t*>(cw + L.leaves);
  int32_t* offsets = reinterpret_cast<int32_t*>(cw + L.offsets);
  int32_t* ext = reinterpret_cast<int32_t*>(cw + L.ext);
  {
    std::vector<int32_t> ex(2 * (size_t)I);
    for (int i = 0; i < I; ++i) {
      ex[2 * i] = p.dev[i % T].pad_h;
      ex[2 * i + 1] = p.dev[i % T].pad_w;
    }
    cudaError_t e0 = cudaMemcpyAsync(ext, ex.data(), ex.size() * 4, cudaMemcpyHostToDevice, st);
    if (e0 == cudaSuccess) e0 = cudaStreamSynchronize(st);   // ex is a host temporary
    if (e0 != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("compressed forward: ") + cudaGetErrorString(e0));
    CompressLay cl;
    ORBIT2_TRY(compress_check(&cc, &cl));
    uint8_t* pw = cw + L.cws_part;
    int passes = 0;
    ORBIT2_TRY(run(c, "compress_partition", st, [&] {
      launch_canny(field, reinterpret_cast<float*>(pw + cl.tmp), reinterpret_cast<float*>(pw + cl.tmp2),
                   reinterpret_cast<float*>(pw + cl.mag), pw + cl.dir, pw + cl.lab,
                   reinterpret_cast<unsigned*>(pw + cl.gmax), reinterpret_cast<int*>(pw + cl.changed), I, L.Hq, L.Wq,
                   cc.sigma, cc.low_frac, cc.high_frac, st, &passes);
      launch_quadtree(pw + cl.lab, reinterpret_cast<int32_t*>(pw + cl.flag), reinterpret_cast<int32_t*>(pw + cl.bsum),
                      offsets + I, leaves, offsets, I, L.Hq, L.Wq, 1, cp->max_side, (double)cc.threshold, st, 0, 0,
                      ext);
      return true;
    }));
  }
  std::vector<int32_t> off(I + 1);
  cudaError_t e = cudaMemcpyAsync(off.data(), offsets, (I + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("compressed forward: ") + cudaGetErrorString(e));
  const int32_t n = off[I];
  if (n_tokens_host) *n_tokens_host = n;
  if (leaves_dev) {
    e = cudaMemcpyAsync(leaves_dev, leaves, (size_t)n * 16, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("compressed forward: ") + cudaGetErrorString(e));
  }
  // 4: tokens (then into the ctx's z: the blocks below use its buffers)
  float* tok = reinterpret_cast<float*>(cw + L.tok);
  ORBIT2_TRY(run(c, "compress_tokens", st, [&] {
    launch_ctokens(z, cd, T, leaves, n, (int)D, e_scale_dev, tok, st);
    return true;
  }));
  e = cudaMemcpyAsync(z, tok, (size_t)n * D * 4, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("compressed forward: ") + cudaGetErrorString(e));
  // the (sample, tile) images as the "tiles" of one call: per image its compressed tokens
  std::vector<DevTile> dt(I + 1);
  std::vector<int32_t> qblk, qpair, qg3;
  int32_t qb = 0, qp = 0;
  for (int b = 0; b <= I; ++b) {
    DevTile t{};
    const int32_t nb = b < I ? off[b + 1] - off[b] : 0;
    t.n_tokens = t.n_core = nb;
    t.tok_off = t.core_off = off[std::min(b, I)];
    t.qb_off = qb;
    t.qp_off = qp;
    t.pad_h = t.core_h = t.out_h = 1;
    t.pad_w = t.core_w = t.out_w = nb;
    dt[b] = t;
    if (b == I) break;
    const int32_t nqb = (nb + 127) / 128;
    for (int32_t i = 0; i < nqb; ++i) qblk.push_back(b);
    for (int32_t i = 0; i < (nqb + 1) / 2; ++i) qpair.push_back(b);
    for (int32_t i = 0; i < nqb; i += 3) qg3.push_back((b << 16) | (i << 2) | (std::min(3, nqb - i) - 1));
    qb += nqb;
    qp += (nqb + 1) / 2;
  }
  if ((int64_t)qblk.size() > L.tabcap || I >= 32768)
    return set_err(ORBIT2_E_CAPACITY, "compressed forward: work-list capacity");
  e = cudaMemcpy(cw + L.tiles, dt.data(), dt.size() * sizeof(DevTile), cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !qblk.empty()) e = cudaMemcpy(cw + L.qblk, qblk.data(), qblk.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !qpair.empty())
    e = cudaMemcpy(cw + L.qpair, qpair.data(), qpair.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && !qg3.empty()) e = cudaMemcpy(cw + L.qg3, qg3.data(), qg3.size() * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("compressed forward tables: ") + cudaGetErrorString(e));
  ChunkDev cc2{};
  cc2.tiles = reinterpret_cast<const DevTile*>(cw + L.tiles);
  cc2.tb = 0; cc2.tc = I; cc2.tok0 = 0; cc2.core0 = 0; cc2.chunk_tokens = n; cc2.chunk_core = n;
  cc2.qb0 = 0; cc2.nqb = qb; cc2.qp0 = 0; cc2.nqp = qp;
  cc2.qblk_tile = reinterpret_cast<const int32_t*>(cw + L.qblk);
  cc2.qpair_tile = reinterpret_cast<const int32_t*>(cw + L.qpair);
  cc2.qpair_core = reinterpret_cast<const int32_t*>(cw + L.qpc);
  cc2.qg3 = reinterpret_cast<const int32_t*>(cw + L.qg3);
  cc2.qg3c = reinterpret_cast<const int32_t*>(cw + L.qg3c);
  cc2.qg0 = 0; cc2.nqg = (int32_t)qg3.size(); cc2.qgc0 = 0; cc2.nqgc = 0; cc2.qc0 = 0; cc2.nqc = 0;
  cc2.core_pairs = 0;
  cc2.core_row = reinterpret_cast<const int32_t*>(cw + L.core_row);
  // 5: the blocks over the compressed tokens (unfused LN; block tail at D = 256)
  const int64_t M = n;
  bf16* xn = c->at<bf16>(ly.xn);
  bf16* qkv = c->at<bf16>(ly.qkv);
  bf16* ao = c->at<bf16>(ly.ao);
  bf16* hid = c->at<bf16>(ly.hid);
  if (mrow > M) {
    e = cudaMemsetAsync(qkv + M * 3 * D, 0, (size_t)(mrow - M) * 3 * D * sizeof(bf16), st);
    if (e != cudaSuccess) return set_err(ORBIT2_E_CUDA, std::string("memset: ") + cudaGetErrorString(e));
  }
  auto gemm = [&](const char* name, int epi, int out_bf, const void* A, int64_t lda, int64_t wo, int64_t nn,
                  int64_t k, EpiParams ep) {
    GemmOperand a{A, mrow, lda, 0}, b{W8 + wo, nn, k};
    ep.M = (int32_t)M;
    ep.N = (int32_t)nn;
    return run(c, name, st, [&] {
      ep.single_cta = c->single_cta_gemm;
      return launch_gemm_tc(epi, out_bf, a, b, M, nn, k, ep, st);
    });
  };
  const bool tail_fused = D == 256;
  for (int l = 0; l < cf.depth && M > 0; ++l) {
    const LayerW& Lw = w.layers[l];
    if (!(tail_fused && l > 0))
      ORBIT2_TRY(run(c, "layernorm", st, [&] {
        launch_layernorm<bf16>(z, wf(Lw.ln1_g), wf(Lw.ln1_b), xn, M, (int)D, nullptr, st);
        return true;
      }));
    EpiParams ep{};
    ep.bias = wf(Lw.b_qkv); ep.C = qkv; ep.ldc = 3 * D;
    ORBIT2_TRY(gemm("qkv_gemm", EPI_BIAS, 1, xn, D, Lw.w_qkv, 3 * D, D, ep));
    ORBIT2_TRY(run(c, "tile_attention", st, [&] {
      return launch_attention_tc(qkv, mrow, ao, cc2, 1, (int)D, cf.heads, p.d, st);
    }));
    if (tail_fused) {
      const bool nxt = l + 1 < cf.depth;
      ORBIT2_TRY(run(c, "block_tail", st, [&] {
        return launch_block_tail(ao, mrow, W8 + Lw.w_o, wf(Lw.b_o), wf(Lw.ln2_g), wf(Lw.ln2_b), W8 + Lw.w_1,
                                 wf(Lw.b_1), W8 + Lw.w_2, wf(Lw.b_2), z, M, (int)D,
                                 nxt ? wf(w.layers[l + 1].ln1_g) : nullptr, nxt ? wf(w.layers[l + 1].ln1_b) : nullptr,
                                 xn, nullptr, 0, st);
      }));
      continue;
    }
    ep = EpiParams{}; ep.bias = wf(Lw.b_o); ep.C = z; ep.ldc = D;
    ORBIT2_TRY(gemm("oproj_gemm", EPI_RESID, 0, ao, D, Lw.w_o, D, D, ep));
    ORBIT2_TRY(run(c, "layernorm", st, [&] {
      launch_layernorm<bf16>(z, wf(Lw.ln2_g), wf(Lw.ln2_b), xn, M, (int)D, nullptr, st);
      return true;
    }));
    ep = EpiParams{}; ep.bias = wf(Lw.b_1); ep.C = hid; ep.ldc = F;
    ORBIT2_TRY(gemm("mlp_up_gemm", EPI_GELU, 1, xn, D, Lw.w_1, F, D, ep));
    ep = EpiParams{}; ep.bias = wf(Lw.b_2); ep.C = z; ep.ldc = D;
    ORBIT2_TRY(gemm("mlp_down_gemm", EPI_RESID, 0, hid, F, Lw.w_2, D, F, ep));
  }
  // 6: LN_f + head per compressed token (the LN output in xn: with halos the tokens can
  // outnumber the core rows hin holds), decompression to the core patches
  bf16* hin = xn;
  bf16* g = reinterpret_cast<bf16*>(cw + L.g);
  if (M > 0) {
    ORBIT2_TRY(run(c, "layernorm", st, [&] {
      launch_layernorm<bf16>(z, wf(w.lnf_g), wf(w.lnf_b), hin, M, (int)D, nullptr, st);
      return true;
    }));
    EpiParams ep{};
    ep.bias = wf(w.b_h); ep.C = g; ep.ldc = p.Nh; ep.M = (int32_t)M; ep.N = p.Nh;
    GemmOperand a{hin, mrow, D, 0}, b{W8 + w.w_h, p.Nh, D};
    ORBIT2_TRY(run(c, "head_gemm", st, [&] {
      ep.single_cta = c->single_cta_gemm;
      return launch_gemm_tc(EPI_BIAS, 1, a, b, M, p.Nh, D, ep, st);
    }));
  }
  return run(c, "decompress", st, [&] {
    launch_decompress(g, cd, T, leaves, n, p.Nh, reinterpret_cast<bf16*>(tile_out_dev), st);
    return true;
  });
}


orbit2_status orbit2_adamw_step(float* w_dev, const float* grad_dev, float* m_dev, float* v_dev, int64_t n,
                                int32_t step, float lr, float beta1, float beta2, float eps, float weight_decay,
                                void* stream) {
  if (n < 0 || step < 1 || !(lr >= 0.f) || !(beta1 >= 0.f && beta1 < 1.f) || !(beta2 >= 0.f && beta2 < 1.f) ||
      !(eps > 0.f))
    return set_err(ORBIT2_E_INVALID, "adamw: n >= 0, step >= 1, lr >= 0, 0 <= beta < 1, eps > 0");
  if (n > 0 && (!w_dev || !grad_dev || !m_dev || !v_dev)) return set_err(ORBIT2_E_INVALID, "adamw: null pointer");
  const double c1 = 1.0 / (1.0 - std::pow((double)beta1, step)), c2 = 1.0 / (1.0 - std::pow((double)beta2, step));
  launch_adamw(w_dev, grad_dev, m_dev, v_dev, n, lr, beta1, beta2, eps, weight_decay, (float)c1, (float)c2,
               reinterpret_cast<cudaStream_t>(stream));
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? ORBIT2_OK : set_err(ORBIT2_E_CUDA, std::string("adamw: ") + cudaGetErrorString(e));
}

}  // extern "C"
