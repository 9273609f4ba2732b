/*
 * orbit2.h -- C ABI of liborbit2.so: the TILES tile-wise, sequence-scaled
 * forward pass of the ORBIT-2 Reslim ViT (arXiv 2505.04802) on B200 (sm_100a).
 *
 * Citations: P:n = PAPER.md line n.  Readings R# = DESIGN.md "Readings".
 *
 * The pass (north star; P:475-498 Reslim, P:511-532 TILES):
 *   (1) split the coarse multi-variable grid into tiles with halo overlap
 *       ("partitions both inputs and downscaled outputs into spatial
 *       tiles"; "each tile is extended with a fixed-width halo");
 *   (2) patch-embed each tile (p = 2);
 *   (3) per-tile multi-head self-attention + MLP blocks (P:527
 *       "self-attention is restricted within each tile");
 *   (4) crop the halos and stitch the tiles into the high-resolution field
 *       ("the halo regions are discarded, and the non-padded tile
 *       outputs are stitched together");
 *   (5) add the residual interpolated upsample of the input.
 * Beyond the pass: the residual / decoder convolutions and the
 * variable aggregation (config fields), the training step (orbit2_train_*,
 * orbit2_loss, orbit2_adamw_step) and the adaptive spatial compression
 * (orbit2_compress_*, orbit2_compressed_forward).
 *
 * Graded boundary: orbit2_tiles_plan (1, host), orbit2_reslim_forward (1-3 +
 * linear head), orbit2_stitch (4-5).  The rest is lifecycle support.
 *
 * Conventions for every call
 *   - Returns orbit2_status; never throws, never aborts, never exits.  On
 *     error, orbit2_last_error() returns a thread-local message naming the
 *     offending field; it stays valid until the next call on that thread.
 *   - Memory: the CALLER allocates and owns every buffer (device buffers are
 *     plain device pointers from cudaMalloc / torch).  The library never
 *     allocates device memory after orbit2_create and never frees caller
 *     memory.  A ctx borrows its workspace until orbit2_destroy.
 *   - Streams: all device work is enqueued on the caller's stream; the forward,
 *     stitch, halo exchange, training forward / loss / backward and weight update
 *     never synchronise the host.  The documented exceptions: orbit2_create
 *     (one-time table upload), orbit2_comm_init / orbit2_comm_status (setup and
 *     status checks), and the data-dependent compression calls orbit2_compress_partition / orbit2_compressed_forward (one
 *     synchronisation per hysteresis pass and one for the token count).
 *     Asynchronous device faults surface at the caller's next synchronisation
 *     (set ORBIT2_SYNC_CHECK=1 to synchronise and check after every call).
 *   - One ctx per host thread / stream at a time.  Distinct ctxs are independent.
 *   - Every device pointer must be 16-byte aligned (TMA / vector access).
 */
#ifndef ORBIT2_H_
#define ORBIT2_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORBIT2_ABI_VERSION 2   /* 2: res_hidden (residual convolutional path) */

typedef enum {
  ORBIT2_OK = 0,
  ORBIT2_E_INVALID = -1,      /* bad argument or configuration (message names the field) */
  ORBIT2_E_CAPACITY = -2,     /* caller buffer / workspace too small (info still filled) */
  ORBIT2_E_UNSUPPORTED = -3,  /* valid but not implemented (e.g. head_dim not in {32,64,128}) */
  ORBIT2_E_CUDA = -4,         /* CUDA runtime / launch error */
  ORBIT2_E_NCCL = -5,         /* reserved (inter-GPU data movement is peer memory, orbit2_comm_*) */
  ORBIT2_E_STATE = -6         /* call made on a ctx in the wrong state */
} orbit2_status;

enum { ORBIT2_HALO_CLAMP = 0, ORBIT2_HALO_REPLICATE = 1 };   /* R4 */
enum { ORBIT2_BF16 = 0, ORBIT2_FP32 = 1 };                   /* arithmetic of the path */

/*
 * Problem statement (north star: "a coarse grid of V variables, a downscale
 * factor, tile size, halo width and ViT width/depth/heads"; P:404 sizes).
 * All extents are in coarse PIXELS except tiles_* (counts) and halo (PATCHES, R3).
 */
typedef struct {
  int32_t abi_version;     /* must be ORBIT2_ABI_VERSION */
  int32_t batch;           /* B >= 1 samples per call */
  int32_t H, W;            /* coarse grid; patch | H, patch | W */
  int32_t V;               /* input variables */
  int32_t K;               /* output variables (1 <= K; K <= V unless out_channel_map) */
  int32_t scale;           /* downscale factor s >= 1 */
  int32_t patch;           /* patch size p (pixels), 1 <= p */
  int32_t tiles_y, tiles_x;/* tile grid; 1 <= tiles_y <= H/p, 1 <= tiles_x <= W/p */
  int32_t halo;            /* halo width in patches, >= 0 */
  int32_t halo_mode;       /* ORBIT2_HALO_CLAMP (default reading R4) or _REPLICATE */
  int32_t embed;           /* D; D % heads == 0, D % 4 == 0, D % 64 == 0 for BF16 */
  int32_t depth;           /* L >= 0 transformer blocks */
  int32_t heads;           /* head_dim = D/heads must be 32, 64 or 128 */
  int32_t mlp_hidden;      /* must be 4*D (R9) */
  int32_t precision;       /* ORBIT2_BF16 or ORBIT2_FP32 */
  int32_t world_size;      /* ranks the tiles are partitioned over (>= 1) */
  int32_t rank;            /* 0 <= rank < world_size */
  int32_t chunk_tiles;     /* max rank-local tiles per forward/stitch call; 0 = all */
  int32_t res_hidden;      /* residual convolutional path (reading R31): hidden
                              channels C_r of res = up + conv_b(GELU(conv_a(up))), 3x3,
                              0 <= C_r <= 64, C_r % 4 == 0; 0 = the bilinear upsample alone */
  int32_t dec_hidden;      /* decoder convolutions (reading R32): hidden channels
                              C_d of conv_db(GELU(conv_da(.))) applied to the
                              unpatchified head output of a tile's core + a ring of
                              ceil(2/P) patches; 0 <= C_d <= 64, C_d % 4 == 0 (needs halo >= that
                              ring); 0 = the linear head alone (R11) */
  int32_t var_agg;         /* 1: per-variable tokens + cross-attention variable
                              aggregation replace the joint patch embedding (P:479,
                              reading R33); 0: joint linear embedding (R1) */
  const int32_t *out_channel_map; /* K entries in [0,V) selecting the residual input
                                     channel of each output variable (R13); NULL = identity */
} orbit2_config;

/* One tile of the plan (R5 uneven split, R6 row-major ids).  Rectangles are
 * half-open, in PATCH units of the coarse patch grid [0,H/p) x [0,W/p). */
typedef struct {
  int32_t tile_id, tile_y, tile_x;  /* tile_id = tile_y * tiles_x + tile_x */
  int32_t owner_rank;               /* rank that computes this tile */
  int32_t local_index;              /* position in owner's rank-local list */
  int32_t core_y0, core_y1, core_x0, core_x1;
  int32_t pad_y0, pad_y1, pad_x0, pad_x1;   /* core +- halo; clipped to the grid
                                               in CLAMP mode, not in REPLICATE */
  int32_t n_tokens;                 /* (pad_y1-pad_y0)*(pad_x1-pad_x0) */
  int32_t n_core_tokens;            /* (core_y1-core_y0)*(core_x1-core_x0) */
  int32_t n_out_tokens;             /* tokens whose head outputs tile_out holds: the core,
                                       grown by ceil(2/P) patches (clipped to the grid)
                                       when dec_hidden > 0 (R32) */
  int64_t token_offset;             /* offset in one sample's packed list of ALL tiles */
  int64_t core_token_offset;        /* offset in one sample's list of ALL core tokens */
} orbit2_tile;

typedef struct {
  int32_t n_tiles;                  /* tiles_y * tiles_x */
  int32_t n_local_tiles;            /* tiles owned by cfg->rank */
  int32_t chunk_tiles;              /* effective max tiles per call */
  int32_t head_dim;
  int64_t tokens_per_sample;        /* sum of n_tokens over all tiles (N_pad) */
  int64_t core_tokens_per_sample;   /* (H/p)*(W/p) */
  int64_t local_tokens;             /* per sample, rank-local tiles */
  int64_t local_core_tokens;        /* per sample, rank-local tiles: OUTPUT tokens (n_out_tokens) */
  int64_t max_chunk_tokens;         /* per sample, max over windows of chunk_tiles local tiles */
  int64_t max_chunk_core_tokens;
  int64_t sum_n2_per_sample;        /* sum_t n_t^2 (attention cost, P:527 O(N^2/T)) */
  int64_t sum_nc_per_sample;        /* sum_t n_t * c_t */
  int64_t workspace_bytes;          /* device workspace needed by orbit2_create */
  int64_t canonical_weight_count;   /* fp32 values in the canonical blob */
  int64_t packed_weight_bytes;      /* device bytes of the packed weights */
  int64_t tile_out_bytes;           /* bytes of tile_out for a full chunk (all B samples) */
  int64_t out_bytes;                /* bytes of out: B*K*(sH)*(sW)*4 */
  double flops_per_sample;          /* algorithmic FLOPs over ALL tiles */
  double local_flops_per_sample;    /* same, rank-local tiles */
  double gather_bytes_per_sample;
  double stitch_bytes_per_sample;
} orbit2_plan_info;

/*
 * orbit2_tiles_plan -- step (1) planning.  Host-only, pure, deterministic; no
 * CUDA calls.  Two-call sizing: tiles = NULL, capacity = 0 fills *info only.
 * If capacity < n_tiles returns ORBIT2_E_CAPACITY with *info filled.
 * Tiles are written in tile_id order.  Ownership: tiles are assigned to ranks
 * by longest-processing-time on the per-tile cost model;
 * rank-local order = increasing tile_id among the rank's tiles.
 * Errors (E_INVALID): p does not divide H or W; tiles_* outside [1, extent/p];
 * halo < 0; embed % heads; embed % 4; mlp_hidden != 4*embed; scale < 1;
 * K < 1; K > V without map; map entry outside [0,V); batch < 1; bad rank.
 * E_UNSUPPORTED: head_dim not in {32,64,128}; BF16 with embed % 64 != 0;
 * BF16 with K*(scale*patch)^2 % 8 != 0 (head-output rows must be 16-byte aligned).
 */
orbit2_status orbit2_tiles_plan(const orbit2_config *cfg, orbit2_tile *tiles,
                                int32_t capacity, orbit2_plan_info *info);

/*
 * orbit2_create -- bind a config to a caller-owned device workspace of at
 * least info.workspace_bytes (from orbit2_tiles_plan).  Uploads the plan
 * tables into the workspace (synchronous, one time).  *ctx receives an
 * opaque handle released by orbit2_destroy.  Uses the current CUDA device.
 */
orbit2_status orbit2_create(const orbit2_config *cfg, void *workspace_dev, size_t workspace_bytes,
                            void **ctx);

/*
 * orbit2_prepare_weights -- convert the canonical fp32 weight blob
 * (canonical_dev, info.canonical_weight_count floats, device memory) into the
 * packed layout the kernels read (packed_dev, info.packed_weight_bytes).
 *
 * Canonical blob (fp32, little endian; PyTorch Linear convention y = W x + b,
 * W stored [out][in] row-major), in this order:
 *   W_e[D][V*p*p] (column (v*p+dy)*p+dx), b_e[D], e_s[D]  (resolution embedding, R8)
 *   per layer l = 0..L-1:
 *     ln1_g[D] ln1_b[D] W_qkv[3D][D] (rows Q|K|V; head h = rows [h*d,(h+1)*d) of each)
 *     b_qkv[3D] W_o[D][D] b_o[D] ln2_g[D] ln2_b[D] W_1[4D][D] b_1[4D] W_2[D][4D] b_2[D]
 *   lnf_g[D] lnf_b[D] W_h[K*P*P][D] (row (k*P+a)*P+b, P = s*p) b_h[K*P*P]
 *   if res_hidden = C_r > 0: W_ra[C_r][K][3][3] b_ra[C_r] W_rb[K][C_r][3][3] b_rb[K]
 *   if dec_hidden = C_d > 0: W_da[C_d][K][3][3] b_da[C_d] W_db[K][C_d][3][3] b_db[K]
 *   if var_agg: W_t[V][D][p*p] e_var[V][D] q_agg[D] W_ak[D][D] b_ak[D] W_av[D][D] b_av[D]
 *               W_ao[D][D] b_ao[D]   (W_e and b_e are then unused)
 * Count = Din*D + 2D + L*(12D^2 + 13D) + 2D + D*K*P^2 + K*P^2 (+ 18 C K + C + K per
 * convolution pair),
 * Din = V*p*p.
 * Stream-ordered; canonical_dev may be freed once the stream passes this call.
 */
orbit2_status orbit2_prepare_weights(void *ctx, const float *canonical_dev, void *packed_dev,
                                     void *stream /* cudaStream_t */);

/*
 * orbit2_reslim_forward -- steps (1)-(3) and the linear decoder head for the
 * rank-local tiles [tile_begin, tile_begin + tile_count) of all B samples.
 *   input_dev : fp32 [B][V][H][W], full-field shaped, row 0 = north.  Read only.
 *               Must hold valid pixels at least inside the padded rects of
 *               the requested tiles.
 *   tile_out_dev : [B][core tokens of the requested tiles, plan order][K*P*P],
 *               bf16 (BF16 path) or fp32 (FP32 path).  Column (k*P+a)*P+b is
 *               output pixel (P*u+a, P*w+b) of variable k for core token (u,w).
 *               Halo tokens produce no output (R16).
 * tile_count <= info.chunk_tiles.  Stream-ordered.
 */
orbit2_status orbit2_reslim_forward(void *ctx, const void *packed_w, const float *input_dev,
                                    int32_t tile_begin, int32_t tile_count, void *tile_out_dev,
                                    void *stream);

/*
 * orbit2_stitch -- steps (4)-(5) for the same tile range: crop (halo outputs
 * were never formed), place the core outputs of tile_out_dev (layout above)
 * into out_dev fp32 [B][K][s*H][s*W], and add the bilinear (align_corners =
 * False, edge clamp; R12) x`s upsample of input channel out_channel_map[k] --
 * with res_hidden > 0 the residual convolutional path up + conv_b(GELU(conv_a(up)))
 * (R31; 3x3, zero padding outside the field; needs input pixels within
 * ceil(2/s) + 1 of the cores, inside the padded rectangles whenever halo >= 1).
 * Writes exactly the output pixels of the requested tiles' cores; other
 * pixels of out_dev are untouched.  Stream-ordered.
 */
orbit2_status orbit2_stitch(void *ctx, const void *tile_out_dev, const float *input_dev,
                            int32_t tile_begin, int32_t tile_count, float *out_dev, void *stream);

/*
 * ---- TILES sequence parallelism across ranks ("assigning each tile to a
 * separate GPU"; "stitched together") ----
 * With world_size = R > 1 each rank computes its LPT-assigned tiles.  Data
 * movement between ranks is expressed as lists of coarse-pixel rectangles
 * (all B samples, all V channels) that the library packs into / unpacks from a
 * contiguous fp32 buffer; the caller moves the buffers (e.g. NCCL send/recv
 * over NVLink).  Message layout: rectangle by rectangle, each [B][V][rows][cols].
 *
 *   ORBIT2_XFER_HALO : halo exchange.  send = pixels of `peer`'s needed tile
 *                      rectangles that lie in this rank's owned cores; recv =
 *                      pixels of this rank's needed rectangles owned by `peer`.
 *                      Needed rectangle of a tile = bounding box of its padded
 *                      rectangle (pixels, clamped to the grid) and its core
 *                      dilated by 1 pixel (the bilinear residual's support, so
 *                      the owner can stitch its tiles; equal to the padded
 *                      rectangle whenever halo >= 1).
 *   ORBIT2_XFER_CORES: input gather to a root.  send = this rank's owned core
 *                      pixels (peer = root); recv (at root) = `peer`'s owned cores.
 * Owned cores: the core rectangles (pixels) of the rank's tiles; they partition
 * the grid.  In CLAMP mode padded rectangles are clipped to the grid; in
 * REPLICATE mode the clamped (edge) pixels are what the gather reads.
 */
typedef struct { int32_t y0, y1, x0, x1; } orbit2_rect;   /* coarse pixels, half-open */
enum { ORBIT2_XFER_HALO = 0, ORBIT2_XFER_CORES = 1 };
enum { ORBIT2_SEND = 0, ORBIT2_RECV = 1 };

/* Host-only, pure: the rectangles and the element count (B*V*sum of areas) of
 * one transfer of cfg->rank with `peer` (peer != rank).  rects may be NULL with
 * cap = 0 (sizing); n_rects receives the count either way; E_CAPACITY if cap
 * is too small. */
orbit2_status orbit2_xfer_plan(const orbit2_config *cfg, int32_t kind, int32_t peer, int32_t direction,
                               orbit2_rect *rects, int32_t cap, int32_t *n_rects, int64_t *n_elems);

/* Pack this rank's SEND rectangles for (kind, peer) from input_dev [B][V][H][W]
 * into buf_dev, or scatter a received buffer into input_dev (RECV rectangles).
 * Stream-ordered; buf_dev holds n_elems floats. */
orbit2_status orbit2_xfer_pack(void *ctx, int32_t kind, int32_t peer, const float *input_dev, float *buf_dev,
                               void *stream);
orbit2_status orbit2_xfer_unpack(void *ctx, int32_t kind, int32_t peer, const float *buf_dev, float *input_dev,
                                 void *stream);

/* Output gather: stitch (steps 4-5, as orbit2_stitch) ALL tiles of rank `peer`
 * from tile_out_dev laid out as that rank's [B][its core tokens, plan order]
 * [K*P*P] (i.e. the tile_out of one orbit2_reslim_forward over all of peer's
 * tiles), reading the residual from input_dev (valid over peer's cores + 1
 * coarse pixel) into out_dev.  peer may equal cfg->rank. */
orbit2_status orbit2_stitch_peer(void *ctx, int32_t peer, const void *tile_out_dev, const float *input_dev,
                                 float *out_dev, void *stream);

/*
 * ---- Peer-memory TILES sequence parallelism (one process per GPU of one
 * NVLink/NVSwitch node; "assigning each tile to a separate GPU"
 * halo, "stitched together").  The library moves the data itself with
 * loads/stores through NVLink peer mappings (CUDA IPC); the caller only swaps
 * the export handles between processes (e.g. torch.distributed all_gather).
 *
 * Per step, on every rank, in stream order:
 *   orbit2_halo_exchange  -- push: the pixels of this rank's owned cores that
 *                            lie in a peer's padded rectangles (plus the 1-pixel
 *                            bilinear support of the peer's cores) are stored
 *                            straight into that peer's input field; then a
 *                            device-side barrier across all ranks.
 *   orbit2_reslim_forward / orbit2_stitch with out_dev = the pointer
 *                            orbit2_comm_target returns: the stitch kernel
 *                            writes this rank's tiles into the gather root's
 *                            output field through NVLink (output gather fused
 *                            into step (4)), or into the local field when
 *                            gather_root = -1 (sharded output).
 *   orbit2_comm_barrier   -- device-side barrier: every rank's stores of this
 *                            step (halo pushes, output tiles) are visible.
 * Precondition of a halo exchange: every rank has passed the previous step's
 * orbit2_comm_barrier (the push overwrites peers' non-owned pixels).
 * Barriers spin on flags in the peers' workspaces with a 30 s timeout; a
 * timeout is reported by orbit2_comm_status (never a hang, never a trap).
 */
typedef struct {
  uint8_t handle[64];   /* cudaIpcMemHandle_t of the allocation holding the buffer */
  int64_t offset;       /* byte offset of the buffer inside that allocation */
  int64_t bytes;        /* allocation size (checked against the plan on open) */
} orbit2_ipc_handle;

/* Host-only: export a device buffer (from cudaMalloc or the torch caching
 * allocator, not from a cudaMallocAsync pool) for the peers of this process. */
orbit2_status orbit2_ipc_export(const void *dev_ptr, orbit2_ipc_handle *out);

/* Collective in the host sense (every rank calls it once, same order):
 * bind the ctx (world_size R, rank r) to
 *   input_dev   this rank's input field [B][V][H][W] fp32 (its owned core pixels
 *               valid before each halo exchange; peers' pushes fill the rest),
 *   out_dev     this rank's output field [B][K][sH][sW] fp32: required on the
 *               gather root and when gather_root = -1 (sharded), else may be NULL,
 *   and every rank's workspace, input field and output field through the R
 *   export handles of each array (entry r = this rank's own, not opened).
 * out_handles may be NULL when gather_root = -1.  Opens the peers' allocations
 * with cudaIpcOpenMemHandle (P2P over NVLink), uploads the push table and
 * zeroes this rank's barrier flags (synchronous; call on every rank before any
 * rank's first halo exchange).  E_STATE if called twice; E_CUDA if a handle
 * cannot be opened; E_INVALID if a peer buffer is smaller than the plan needs. */
orbit2_status orbit2_comm_init(void *ctx, int32_t gather_root, float *input_dev, float *out_dev,
                               const orbit2_ipc_handle *workspace_handles, const orbit2_ipc_handle *input_handles,
                               const orbit2_ipc_handle *out_handles);

/* The output field this rank's orbit2_stitch calls write: the gather root's
 * field mapped into this process, or out_dev of orbit2_comm_init on the root
 * and when the output is sharded (gather_root = -1). */
orbit2_status orbit2_comm_target(void *ctx, float **out_dev);

/* Halo push of this step (all B samples, all V channels) + barrier slot 0. */
orbit2_status orbit2_halo_exchange(void *ctx, void *stream);
/* End-of-step barrier (slot 1): every rank's earlier stores are visible. */
orbit2_status orbit2_comm_barrier(void *ctx, void *stream);

/* Synchronises the device and reports a barrier timeout (E_STATE, the message
 * names the missing rank) or a CUDA error; OK otherwise. */
orbit2_status orbit2_comm_status(void *ctx);

/* Number of kernels the library launched on this ctx so far. */
/* ==========================================================================
 * Training step.  The paper's throughput numbers are
 * training numbers ("Only the mixed-precision BFLOAT16 results"); the step is
 *   out = TILES forward (every query of every block kept for the backward)
 *   L   = Bayesian loss (readings R34, R35): per sample
 *         (1/(K N)) [ sum_i w_row(i) (y_i - x_i)^2 + lambda sum_i sum_{j in C(i)} b_ij h(x_i - x_j) ],
 *         C(i) the 8 neighbours inside the field, b_ij = 1/euclidean distance,
 *         h the Huber-smoothed |.| with width delta, w_row = cos(lat) / mean cos(lat)
 *         (geo != 0; else 1); the batch loss is the mean over the B samples
 *   dL/dweights by reverse-mode differentiation of the tiled forward, written into a
 *         caller buffer in the CANONICAL blob order (fp32, same count), for the
 *         rank-local tiles (summing the ranks' gradients, or averaging data-parallel
 *         replicas' with one all-reduce, is the caller's once-per-batch step, R36)
 * Scope (E_UNSUPPORTED otherwise): BF16 precision, head_dim 64, embed <= 1024,
 * var_agg = res_hidden = dec_hidden = 0, one call over every rank-local tile.
 * The oracle is oracle/train.py.
 * ========================================================================== */
typedef struct {
  int64_t workspace_bytes;          /* device bytes orbit2_train_bind needs: the activations
                                       every block keeps for the backward, the backward's
                                       scratch and transposed bf16 weights */
  int64_t canonical_weight_count;   /* fp32 values of the gradient (= the canonical blob) */
  double fwd_flops_per_sample;      /* training forward, rank-local tiles */
  double flops_per_sample;          /* forward + backward algorithmic FLOPs, rank-local tiles */
  double attn_bwd_flops_per_sample; /* attention backward alone (S, dP, dV, dK, dQ) */
} orbit2_train_info;

/* Sizing (host only). */
orbit2_status orbit2_train_plan(void *ctx, orbit2_train_info *info);
/* Bind a caller-owned device buffer of >= info.workspace_bytes (16-byte aligned) to the
 * context; zero-fills it on `stream` (rows past the batch's tokens must stay zero). */
orbit2_status orbit2_train_bind(void *ctx, void *train_ws_dev, size_t bytes, void *stream);
/* Transposed bf16 copies of the weights the input-gradient GEMMs read, from the
 * canonical fp32 blob; call after every weight update (with orbit2_prepare_weights). */
orbit2_status orbit2_train_prepare(void *ctx, const float *canonical_dev, void *stream);
/* Forward over every rank-local tile (steps 1-3 + head, all queries of every block),
 * keeping the activations in the training workspace; tile_out as orbit2_reslim_forward.
 * The output field is then assembled by orbit2_stitch as for inference. */
orbit2_status orbit2_train_forward(void *ctx, const void *packed_w, const float *input_dev,
                                   void *tile_out_dev, void *stream);
/* Bayesian loss of out_dev [B][K][sH][sW] against truth_dev (same shape), fp32:
 * loss_dev[b] (double, per sample, overwritten) and dout_dev = d(mean_b loss_b)/d out
 * (fp32, same shape, overwritten).  delta > 0, lambda >= 0 (E_INVALID otherwise). */
orbit2_status orbit2_loss(void *ctx, const float *out_dev, const float *truth_dev, float lambda, float delta,
                          int32_t geo, double *loss_dev, float *dout_dev, void *stream);
/* Backward of the last orbit2_train_forward given dout_dev [B][K][sH][sW] (the stitch
 * read backwards: only the rank-local tiles' core pixels are read).  grad_dev
 * (canonical order, info.canonical_weight_count floats, 16-byte aligned) is
 * overwritten with the gradient of the rank-local tiles' contribution. */
orbit2_status orbit2_train_backward(void *ctx, const void *packed_w, const float *dout_dev, float *grad_dev,
                                    void *stream);
/* The weight update (the paper names no optimizer; reading R43: AdamW, decoupled weight decay,
 * bias-corrected moments), elementwise over n fp32 values in place: m, v (caller-owned, zero
 * before step 1) and w (the canonical blob).  step = t >= 1.  Re-run orbit2_prepare_weights and
 * orbit2_train_prepare on the updated blob before the next step. */
orbit2_status orbit2_adamw_step(float *w_dev, const float *grad_dev, float *m_dev, float *v_dev, int64_t n,
                                int32_t step, float lr, float beta1, float beta2, float eps, float weight_decay,
                                void *stream);

/* ==========================================================================
 * Adaptive spatial compression (readings R37-R40).
 * "the model projects the embedding back into image space and recursively partitions it
 * into spatial quadrants using a quad-tree structure.  Partitioning continues for any
 * quadrant where the estimated feature density -- computed via Canny edge detection --
 * exceeds a predefined threshold, terminating when a minimum patch size is reached"
 * (P:483).  Context-free calls on caller-owned device buffers; the oracle is
 * oracle/compress.py.  Fields are [B][H][W] (partition) / [B][C][H][W] (features), with H, W
 * multiples of max_side (pad by edge replication first); max_side = min_side * 2^k,
 * 1 <= k <= 6; sigma in (0, 8/3]; 0 < low_frac <= high_frac.
 * ========================================================================== */
typedef struct {
  int32_t batch;            /* B fields */
  int32_t H, W;             /* pixels */
  int32_t C;                /* feature channels (tokenize / detokenize) */
  int32_t min_side;         /* the smallest leaf = the token's pooled size m (pixels) */
  int32_t max_side;         /* the quad-tree root cells */
  int32_t embed;            /* D: token width */
  float threshold;          /* split iff edge pixels / area > threshold (R38); < 0: split to min_side */
  float sigma, low_frac, high_frac;   /* Canny (R37) */
} orbit2_compress_config;

/* Sizing (host only): device workspace bytes of orbit2_compress_partition and the
 * capacity of the leaf list (B * (H/min_side) * (W/min_side)). */
orbit2_status orbit2_compress_plan(const orbit2_compress_config *cfg, int64_t *workspace_bytes,
                                   int64_t *max_patches);
/* Canny edge map + quad-tree of every field: patches_dev [max_patches][4] int32 receives the
 * leaves (image, row, col, side) in (image, row, col) order, offsets_dev [B + 1] the first
 * leaf of every image (offsets[B] = total), *n_host the total (the call synchronises the
 * stream once per hysteresis pass: the leaf count is data-dependent).  edges_dev (nullable,
 * [B][H][W] uint8) receives the edge map (1 = edge). */
orbit2_status orbit2_compress_partition(const orbit2_compress_config *cfg, const float *image_dev,
                                        void *workspace_dev, size_t workspace_bytes, uint8_t *edges_dev,
                                        int32_t *patches_dev, int32_t *offsets_dev, int32_t *n_host,
                                        void *stream);
/* tokens_dev [n][D] = W_tok pool(leaf) + b_tok + e_scale[log2(side / min_side)]; w_tok
 * [D][C m m] (column (c m + i) m + j), b_tok [D], e_scale [k + 1][D] (R39).  One fp32 GEMM
 * over all leaves (the scale embedding on one-hot columns); workspace as planned. */
orbit2_status orbit2_compress_tokenize(const orbit2_compress_config *cfg, void *workspace_dev, size_t workspace_bytes,
                                       const float *feat_dev, const int32_t *patches_dev, int32_t n,
                                       const float *w_tok, const float *b_tok, const float *e_scale,
                                       float *tokens_dev, void *stream);
/* out_dev [B][C][H][W] = smooth(broadcast(W_dec t + b_dec)); w_dec [C m m][D], b_dec [C m m],
 * w_sm [C][C][3][3], b_sm [C]; work_dev: [B][C][H][W] scratch (R40). */
orbit2_status orbit2_compress_detokenize(const orbit2_compress_config *cfg, void *workspace_dev,
                                         size_t workspace_bytes, const float *tokens_dev,
                                         const int32_t *patches_dev, int32_t n, const float *w_dec,
                                         const float *b_dec, const float *w_sm, const float *b_sm,
                                         float *work_dev, float *out_dev, void *stream);

/* The Reslim forward on compressed tokens (R41, R42), per (sample, tile) "image" i = b T + t
 * of the T rank-local tiles: z0 = the patch embedding of every patch of the tile's padded
 * rectangle (O2, O3); the compression field = z0 averaged over its D channels, edge-padded
 * to one shape for all tiles (the largest padded rectangle rounded up to max_side); leaves =
 * orbit2_compress_partition of that field with min_side = 1 patch (leaves rooted outside
 * the rectangle dropped); token = mean of z0 over the leaf's rectangle patches +
 * e_scale[log2 side]; the ViT blocks attend over each image's tokens (attention stays in the
 * tile); LN_f + head per token; every CORE patch of a leaf gets its token's head
 * output in tile_out ([B][core tokens of all local tiles][K P^2] bf16, the layout of
 * orbit2_reslim_forward over every local tile), which orbit2_stitch turns into the field
 * (the halo is discarded).  The context must be BF16 with one call over every
 * rank-local tile (chunk_tiles = 0), without var_agg / dec_hidden / res_hidden
 * (E_UNSUPPORTED otherwise).  Synchronises the stream once per hysteresis pass and once for
 * the token count. */
typedef struct {
  int32_t max_side;         /* quad-tree root cells (patches), a power of two >= 2 */
  float threshold, sigma, low_frac, high_frac;   /* R37 / R38 */
} orbit2_compression;
/* workspace bytes of orbit2_compressed_forward; *levels = log2(max_side) + 1 rows of e_scale */
orbit2_status orbit2_compressed_plan(void *ctx, const orbit2_compression *cp, int64_t *workspace_bytes,
                                     int32_t *levels);
/* e_scale_dev [levels][D] fp32; leaves_dev (nullable) receives the leaves [n][4] (image
 * b T + t, u0, w0 in the tile's padded rectangle, side; patches); *n_tokens_host the count. */
orbit2_status orbit2_compressed_forward(void *ctx, const void *packed_w, const float *input_dev,
                                        const orbit2_compression *cp, const float *e_scale_dev, void *workspace_dev,
                                        size_t workspace_bytes, void *tile_out_dev, int32_t *leaves_dev,
                                        int32_t *n_tokens_host, void *stream);

int64_t orbit2_launch_count(void *ctx);

/*
 * Per-kernel-class timing with CUDA events on the call's stream.  When
 * enabled, every launch is bracketed by events; orbit2_kernel_times() then
 * synchronises the last event and returns, for up to `cap` classes, the name,
 * the number of launches and the summed device milliseconds since the last
 * reset.  Returns the number of classes.  Not for timed throughput runs.
 */
orbit2_status orbit2_set_profiling(void *ctx, int32_t enable);
int32_t orbit2_kernel_times(void *ctx, const char **names, int64_t *launches, double *ms,
                            int32_t cap);

const char *orbit2_last_error(void);
void orbit2_destroy(void *ctx);

#ifdef __cplusplus
}
#endif
#endif /* ORBIT2_H_ */
