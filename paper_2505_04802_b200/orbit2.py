"""Thin ctypes binding of liborbit2.so (include/orbit2.h).

Argument marshalling only: every step of the pass runs in the library's
kernels.  PyTorch supplies device memory and streams.  There is no CPU
fallback: if the library is missing or fails to load, importing this module
raises.
"""
from __future__ import annotations

import ctypes as C

_ct = C   # ctypes under a name no parameter shadows
import os

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ORBIT2_LIB") or os.path.join(PKG, "liborbit2.so")   # ORBIT2_LIB: A/B builds

ABI_VERSION = 2
OK, E_INVALID, E_CAPACITY, E_UNSUPPORTED, E_CUDA, E_NCCL, E_STATE = 0, -1, -2, -3, -4, -5, -6
HALO_CLAMP, HALO_REPLICATE = 0, 1
BF16, FP32 = 0, 1
XFER_HALO, XFER_CORES = 0, 1
SEND, RECV = 0, 1


class orbit2_config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "abi_version", "batch", "H", "W", "V", "K", "scale", "patch", "tiles_y", "tiles_x", "halo",
        "halo_mode", "embed", "depth", "heads", "mlp_hidden", "precision", "world_size", "rank",
        "chunk_tiles", "res_hidden", "dec_hidden", "var_agg")] + [("out_channel_map", C.POINTER(C.c_int32))]


class orbit2_tile(C.Structure):
    _fields_ = [(n, C.c_int32) for n in (
        "tile_id", "tile_y", "tile_x", "owner_rank", "local_index", "core_y0", "core_y1", "core_x0",
        "core_x1", "pad_y0", "pad_y1", "pad_x0", "pad_x1", "n_tokens", "n_core_tokens", "n_out_tokens")] + [
        ("token_offset", C.c_int64), ("core_token_offset", C.c_int64)]


class orbit2_plan_info(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n_tiles", "n_local_tiles", "chunk_tiles", "head_dim")] + [
        (n, C.c_int64) for n in (
            "tokens_per_sample", "core_tokens_per_sample", "local_tokens", "local_core_tokens",
            "max_chunk_tokens", "max_chunk_core_tokens", "sum_n2_per_sample", "sum_nc_per_sample",
            "workspace_bytes", "canonical_weight_count", "packed_weight_bytes", "tile_out_bytes",
            "out_bytes")] + [(n, C.c_double) for n in (
                "flops_per_sample", "local_flops_per_sample", "gather_bytes_per_sample",
                "stitch_bytes_per_sample")]


class orbit2_train_info(C.Structure):
    _fields_ = [("workspace_bytes", C.c_int64), ("canonical_weight_count", C.c_int64),
                ("fwd_flops_per_sample", C.c_double), ("flops_per_sample", C.c_double),
                ("attn_bwd_flops_per_sample", C.c_double)]


class orbit2_compress_config(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("batch", "H", "W", "C", "min_side", "max_side", "embed")] + [
        (n, C.c_float) for n in ("threshold", "sigma", "low_frac", "high_frac")]


class orbit2_compression(C.Structure):
    _fields_ = [("max_side", C.c_int32)] + [(n, C.c_float) for n in ("threshold", "sigma", "low_frac", "high_frac")]


class orbit2_rect(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("y0", "y1", "x0", "x1")]


class orbit2_ipc_handle(C.Structure):
    _fields_ = [("handle", C.c_uint8 * 64), ("offset", C.c_int64), ("bytes", C.c_int64)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2505_04802_b200.build` "
                          "(there is no CPU fallback)")
    lib = C.CDLL(LIB_PATH)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "orbit2_tiles_plan": (i32, [C.POINTER(orbit2_config), C.POINTER(orbit2_tile), i32,
                                    C.POINTER(orbit2_plan_info)]),
        "orbit2_create": (i32, [C.POINTER(orbit2_config), vp, C.c_size_t, C.POINTER(vp)]),
        "orbit2_prepare_weights": (i32, [vp, vp, vp, vp]),
        "orbit2_reslim_forward": (i32, [vp, vp, vp, i32, i32, vp, vp]),
        "orbit2_stitch": (i32, [vp, vp, vp, i32, i32, vp, vp]),
        "orbit2_xfer_plan": (i32, [C.POINTER(orbit2_config), i32, i32, i32, C.POINTER(orbit2_rect), i32,
                                   C.POINTER(i32), C.POINTER(i64)]),
        "orbit2_xfer_pack": (i32, [vp, i32, i32, vp, vp, vp]),
        "orbit2_xfer_unpack": (i32, [vp, i32, i32, vp, vp, vp]),
        "orbit2_stitch_peer": (i32, [vp, i32, vp, vp, vp, vp]),
        "orbit2_ipc_export": (i32, [vp, C.POINTER(orbit2_ipc_handle)]),
        "orbit2_comm_init": (i32, [vp, i32, vp, vp, C.POINTER(orbit2_ipc_handle), C.POINTER(orbit2_ipc_handle),
                                   C.POINTER(orbit2_ipc_handle)]),
        "orbit2_comm_target": (i32, [vp, C.POINTER(vp)]),
        "orbit2_halo_exchange": (i32, [vp, vp]),
        "orbit2_comm_barrier": (i32, [vp, vp]),
        "orbit2_comm_status": (i32, [vp]),
        "orbit2_train_plan": (i32, [vp, C.POINTER(orbit2_train_info)]),
        "orbit2_train_bind": (i32, [vp, vp, C.c_size_t, vp]),
        "orbit2_train_prepare": (i32, [vp, vp, vp]),
        "orbit2_train_forward": (i32, [vp, vp, vp, vp, vp]),
        "orbit2_loss": (i32, [vp, vp, vp, C.c_float, C.c_float, i32, vp, vp, vp]),
        "orbit2_train_backward": (i32, [vp, vp, vp, vp, vp]),
        "orbit2_adamw_step": (i32, [vp, vp, vp, vp, i64, i32, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float,
                                    vp]),
        "orbit2_compress_plan": (i32, [C.POINTER(orbit2_compress_config), C.POINTER(i64), C.POINTER(i64)]),
        "orbit2_compress_partition": (i32, [C.POINTER(orbit2_compress_config), vp, vp, C.c_size_t, vp, vp, vp,
                                            C.POINTER(i32), vp]),
        "orbit2_compress_tokenize": (i32, [C.POINTER(orbit2_compress_config), vp, C.c_size_t, vp, vp, i32, vp,
                                           vp, vp, vp, vp]),
        "orbit2_compress_detokenize": (i32, [C.POINTER(orbit2_compress_config), vp, C.c_size_t, vp, vp, i32, vp,
                                             vp, vp, vp, vp, vp, vp]),
        "orbit2_compressed_plan": (i32, [vp, C.POINTER(orbit2_compression), C.POINTER(i64), C.POINTER(i32)]),
        "orbit2_compressed_forward": (i32, [vp, vp, vp, C.POINTER(orbit2_compression), vp, vp, C.c_size_t, vp, vp,
                                            C.POINTER(i32), vp]),
        "orbit2_launch_count": (i64, [vp]),
        "orbit2_set_profiling": (i32, [vp, i32]),
        "orbit2_kernel_times": (i32, [vp, C.POINTER(C.c_char_p), C.POINTER(i64), C.POINTER(C.c_double), i32]),
        "orbit2_last_error": (C.c_char_p, []),
        "orbit2_destroy": (None, [vp]),
    }
    for name, (res, args) in sig.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    return lib


lib = _load()
EXPORTED = ("orbit2_tiles_plan", "orbit2_create", "orbit2_prepare_weights", "orbit2_reslim_forward",
            "orbit2_stitch", "orbit2_xfer_plan", "orbit2_xfer_pack", "orbit2_xfer_unpack", "orbit2_stitch_peer",
            "orbit2_ipc_export", "orbit2_comm_init", "orbit2_comm_target", "orbit2_halo_exchange",
            "orbit2_comm_barrier", "orbit2_comm_status",
            "orbit2_train_plan", "orbit2_train_bind", "orbit2_train_prepare", "orbit2_train_forward",
            "orbit2_loss", "orbit2_train_backward", "orbit2_adamw_step",
            "orbit2_compress_plan", "orbit2_compress_partition", "orbit2_compress_tokenize",
            "orbit2_compress_detokenize", "orbit2_compressed_plan", "orbit2_compressed_forward",
            "orbit2_launch_count", "orbit2_set_profiling", "orbit2_kernel_times", "orbit2_last_error",
            "orbit2_destroy")


class Orbit2Error(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib.orbit2_last_error().decode()
        super().__init__(f"{where} failed with status {status}: {msg}")
        self.status = status


def _check(st: int, where: str):
    if st != OK:
        raise Orbit2Error(st, where)


def make_config(*, H, W, V, K, scale, patch, tiles_y, tiles_x, halo, embed, depth, heads, batch=1,
                halo_mode=HALO_CLAMP, precision=BF16, world_size=1, rank=0, chunk_tiles=0,
                out_channel_map=None, res_hidden=0, dec_hidden=0, var_agg=0) -> orbit2_config:
    """Build an orbit2_config (the paper's problem statement, north star)."""
    cfg = orbit2_config(ABI_VERSION, batch, H, W, V, K, scale, patch, tiles_y, tiles_x, halo, halo_mode,
                        embed, depth, heads, 4 * embed, precision, world_size, rank, chunk_tiles, res_hidden,
                        dec_hidden, var_agg, None)
    if out_channel_map is not None:
        arr = (C.c_int32 * K)(*out_channel_map)
        cfg.out_channel_map = C.cast(arr, C.POINTER(C.c_int32))
        cfg._map_keepalive = arr
    return cfg


def config_from(w, **over) -> orbit2_config:
    """orbit2_config from any object with the workload fields (e.g. workloads.Config)."""
    kw = dict(H=w.H, W=w.W, V=w.V, K=w.K, scale=w.scale, patch=w.patch, tiles_y=w.tiles_y,
              tiles_x=w.tiles_x, halo=w.halo, embed=w.embed, depth=w.depth, heads=w.heads,
              batch=w.batch, halo_mode=w.halo_mode, out_channel_map=w.out_channel_map,
              res_hidden=getattr(w, "res_hidden", 0), dec_hidden=getattr(w, "dec_hidden", 0),
              var_agg=getattr(w, "var_agg", 0))
    kw.update(over)
    return make_config(**kw)


def config_from_cfg(cfg: orbit2_config, **over) -> orbit2_config:
    """Copy of an orbit2_config with fields replaced (e.g. rank=peer)."""
    new = orbit2_config()
    C.pointer(new)[0] = cfg
    for k, v in over.items():
        setattr(new, k, v)
    if hasattr(cfg, "_map_keepalive"):
        new._map_keepalive = cfg._map_keepalive
    return new


def orbit2_tiles_plan(cfg: orbit2_config):
    """Step (1) planning (host only).  Returns (list of orbit2_tile, orbit2_plan_info)."""
    info = orbit2_plan_info()
    _check(lib.orbit2_tiles_plan(C.byref(cfg), None, 0, C.byref(info)), "orbit2_tiles_plan(size)")
    tiles = (orbit2_tile * info.n_tiles)()
    _check(lib.orbit2_tiles_plan(C.byref(cfg), tiles, info.n_tiles, C.byref(info)), "orbit2_tiles_plan")
    return list(tiles), info


def orbit2_xfer_plan(cfg: orbit2_config, kind: int, peer: int, direction: int):
    """Rectangles (coarse pixels) and element count of one rank-to-rank transfer (host only)."""
    n = C.c_int32()
    e = C.c_int64()
    _check(lib.orbit2_xfer_plan(C.byref(cfg), kind, peer, direction, None, 0, C.byref(n), C.byref(e)),
           "orbit2_xfer_plan(size)")
    rects = (orbit2_rect * max(n.value, 1))()
    _check(lib.orbit2_xfer_plan(C.byref(cfg), kind, peer, direction, rects, n.value, C.byref(n), C.byref(e)),
           "orbit2_xfer_plan")
    return [(r.y0, r.y1, r.x0, r.x1) for r in rects[:n.value]], int(e.value)


def _ptr(t) -> int:
    return t.data_ptr()


def _req(t, dtype, name):
    """The ABI takes raw pointers: check what the C side cannot (dtype, device,
    contiguity) so a float64 or strided tensor fails here instead of being
    reinterpreted."""
    if not t.is_cuda or t.dtype != dtype or not t.is_contiguous():
        raise TypeError(f"{name}: expected a contiguous CUDA {dtype} tensor, got {t.dtype} "
                        f"on {t.device} (contiguous={t.is_contiguous()})")
    return t


def _stream(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


class _on_device:
    """Run a library call with the ctx's device current (kernel attributes, SM
    counts and launches are per device)."""

    def __init__(self, dev):
        self.dev = dev

    def __enter__(self):
        import torch
        self.prev = torch.cuda.current_device()
        if self.prev != self.dev.index:
            torch.cuda.set_device(self.dev)

    def __exit__(self, *a):
        import torch
        if self.prev != self.dev.index:
            torch.cuda.set_device(self.prev)


class Context:
    """One orbit2 ctx bound to a torch-allocated workspace on the current device."""

    def __init__(self, cfg: orbit2_config, device=None):
        import torch
        self.cfg = cfg
        self.tiles, self.info = orbit2_tiles_plan(cfg)
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.workspace = torch.empty(max(self.info.workspace_bytes, 16), dtype=torch.uint8, device=self.device)
        if os.environ.get("ORBIT2_POISON_WORKSPACE") == "1":   # tests: NaN bytes expose reads of unwritten rows
            self.workspace.fill_(0xFF)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            _check(lib.orbit2_create(C.byref(cfg), _ptr(self.workspace), self.info.workspace_bytes, C.byref(h)),
                   "orbit2_create")
        self.handle = h
        self.bf16 = cfg.precision == BF16
        self.sH, self.sW = cfg.scale * cfg.H, cfg.scale * cfg.W

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value and lib is not None:
            lib.orbit2_destroy(h)
            self.handle = None

    # -- lifecycle ---------------------------------------------------------
    def prepare_weights(self, canonical_dev, stream=None, out=None):
        """Pack the canonical fp32 blob (into `out` when given: re-packing after a weight update)."""
        import torch
        assert canonical_dev.dtype == torch.float32 and canonical_dev.is_cuda
        assert canonical_dev.numel() == self.info.canonical_weight_count, "canonical blob size"
        packed = torch.empty(self.info.packed_weight_bytes, dtype=torch.uint8, device=self.device) if out is None \
            else out
        with _on_device(self.device):
            _check(lib.orbit2_prepare_weights(self.handle, _ptr(canonical_dev), _ptr(packed), _stream(stream)),
                   "orbit2_prepare_weights")
        return packed

    def tile_out_buffer(self, tile_count=None):
        import torch
        info = self.info
        dt = torch.bfloat16 if self.bf16 else torch.float32
        nh = self.cfg.K * (self.cfg.scale * self.cfg.patch) ** 2
        return torch.empty((self.cfg.batch * info.max_chunk_core_tokens, nh), dtype=dt, device=self.device)

    # -- the graded calls --------------------------------------------------
    def orbit2_reslim_forward(self, packed, x_dev, tile_begin, tile_count, tile_out, stream=None):
        import torch
        _req(x_dev, torch.float32, "x_dev")
        _req(tile_out, torch.bfloat16 if self.bf16 else torch.float32, "tile_out")
        with _on_device(self.device):
            _check(lib.orbit2_reslim_forward(self.handle, _ptr(packed), _ptr(x_dev), tile_begin, tile_count,
                                             _ptr(tile_out), _stream(stream)), "orbit2_reslim_forward")

    def orbit2_stitch(self, tile_out, x_dev, tile_begin, tile_count, out, stream=None):
        import torch
        _req(x_dev, torch.float32, "x_dev")
        _req(out, torch.float32, "out")
        _req(tile_out, torch.bfloat16 if self.bf16 else torch.float32, "tile_out")
        with _on_device(self.device):
            _check(lib.orbit2_stitch(self.handle, _ptr(tile_out), _ptr(x_dev), tile_begin, tile_count, _ptr(out),
                                     _stream(stream)), "orbit2_stitch")

    def _stitch_to(self, tile_out, x_dev, tile_begin, tile_count, out_ptr: int, stream=None):
        """orbit2_stitch into a raw device address (a peer's field mapped into this
        process, from comm_target())."""
        import torch
        _req(x_dev, torch.float32, "x_dev")
        _req(tile_out, torch.bfloat16 if self.bf16 else torch.float32, "tile_out")
        with _on_device(self.device):
            _check(lib.orbit2_stitch(self.handle, _ptr(tile_out), _ptr(x_dev), tile_begin, tile_count, out_ptr,
                                     _stream(stream)), "orbit2_stitch")

    # -- peer-memory TILES sequence parallelism (orbit2_comm_*) ---------------
    def ipc_handles(self, x_dev, out_dev):
        """Export handles of this rank's workspace, input field and output field
        (None -> zero handle) as raw bytes, for the all-gather between processes."""
        def one(t):
            h = orbit2_ipc_handle()
            if t is not None:
                _check(lib.orbit2_ipc_export(_ptr(t), C.byref(h)), "orbit2_ipc_export")
            return bytes(h)
        return one(self.workspace), one(x_dev), one(out_dev)

    def comm_init(self, gather_root, x_dev, out_dev, handles):
        """handles: per rank (workspace, input, output) export bytes, rank order."""
        R = self.cfg.world_size
        if len(handles) != R:
            raise ValueError("comm_init: one handle triple per rank")
        arrs = [(orbit2_ipc_handle * R)() for _ in range(3)]
        for r, trip in enumerate(handles):
            for a, b in zip(arrs, trip):
                C.memmove(C.byref(a[r]), b, C.sizeof(orbit2_ipc_handle))
        with _on_device(self.device):
            _check(lib.orbit2_comm_init(self.handle, gather_root, _ptr(x_dev),
                                        _ptr(out_dev) if out_dev is not None else None, arrs[0], arrs[1], arrs[2]),
                   "orbit2_comm_init")
        p = C.c_void_p()
        _check(lib.orbit2_comm_target(self.handle, C.byref(p)), "orbit2_comm_target")
        return p.value

    def halo_exchange(self, stream=None):
        with _on_device(self.device):
            _check(lib.orbit2_halo_exchange(self.handle, _stream(stream)), "orbit2_halo_exchange")

    def comm_barrier(self, stream=None):
        with _on_device(self.device):
            _check(lib.orbit2_comm_barrier(self.handle, _stream(stream)), "orbit2_comm_barrier")

    def comm_status(self):
        with _on_device(self.device):
            _check(lib.orbit2_comm_status(self.handle), "orbit2_comm_status")

    # -- multi-rank (TILES sequence parallelism) ------------------------------
    def orbit2_xfer_pack(self, kind, peer, x_dev, buf, stream=None):
        _check(lib.orbit2_xfer_pack(self.handle, kind, peer, _ptr(x_dev), _ptr(buf), _stream(stream)),
               "orbit2_xfer_pack")

    def orbit2_xfer_unpack(self, kind, peer, buf, x_dev, stream=None):
        _check(lib.orbit2_xfer_unpack(self.handle, kind, peer, _ptr(buf), _ptr(x_dev), _stream(stream)),
               "orbit2_xfer_unpack")

    def orbit2_stitch_peer(self, peer, tile_out, x_dev, out, stream=None):
        _check(lib.orbit2_stitch_peer(self.handle, peer, _ptr(tile_out), _ptr(x_dev), _ptr(out), _stream(stream)),
               "orbit2_stitch_peer")

    def rank_tile_out(self):
        """tile_out covering ALL of this rank's tiles: [B][local core tokens][K*P*P]."""
        import torch
        nh = self.cfg.K * (self.cfg.scale * self.cfg.patch) ** 2
        dt = torch.bfloat16 if self.bf16 else torch.float32
        return torch.empty((self.cfg.batch * max(self.info.local_core_tokens, 1), nh), dtype=dt, device=self.device)

    def forward_rank(self, packed, x_dev, tile_out, stream=None):
        """Steps (1)-(3) + head over all of this rank's tiles into a rank-wide
        tile_out (chunked calls write consecutive slices: needs B == 1 when
        chunk_tiles < n_local_tiles)."""
        n, ch = self.info.n_local_tiles, self.info.chunk_tiles
        if n == 0:                      # a rank that owns no tiles (world_size > n_tiles)
            return tile_out
        if ch < n and self.cfg.batch != 1:
            raise ValueError("rank-wide tile_out with chunked calls needs batch == 1")
        nh = tile_out.shape[1]
        for tb in range(0, n, ch):
            tc = min(ch, n - tb)
            off = self.tiles_core_offset(tb)
            self.orbit2_reslim_forward(packed, x_dev, tb, tc, tile_out[off:], stream)
        return tile_out

    def tiles_core_offset(self, tb):
        """Core-token offset (one sample) of rank-local tile tb."""
        if not hasattr(self, "_core_off"):
            r = self.cfg.rank
            mine = [t for t in self.tiles if t.owner_rank == r]
            offs, acc = [], 0
            for t in mine:
                offs.append(acc)
                acc += t.n_out_tokens
            offs.append(acc)
            self._core_off = offs
        return self._core_off[tb]

    # -- convenience: all rank-local tiles, chunk by chunk ------------------
    def forward(self, packed, x_dev, out=None, tile_out=None, stream=None):
        import torch
        cfg = self.cfg
        if out is None:
            out = torch.empty((cfg.batch, cfg.K, self.sH, self.sW), dtype=torch.float32, device=self.device)
        if tile_out is None:
            tile_out = self.tile_out_buffer()
        n, ch = self.info.n_local_tiles, self.info.chunk_tiles
        for tb in range(0, n, max(ch, 1)):      # no iterations for a rank without tiles
            tc = min(ch, n - tb)
            self.orbit2_reslim_forward(packed, x_dev, tb, tc, tile_out, stream)
            self.orbit2_stitch(tile_out, x_dev, tb, tc, out, stream)
        return out

    # -- host buffers in, host buffers out (pipelined) ------------------------
    def forward_host(self, packed, x_host, out_host, stream=None, sync_out=True):
        """The whole pass for N = k * cfg.batch samples held in PINNED host memory:
        x_host [N,V,H,W] fp32 -> out_host [N,K,sH,sW] fp32.  Samples go through the
        device in groups of cfg.batch; the host->device copy of group g+1 and the
        device->host copy of group g-1 run on their own streams (copy engines, both
        PCIe directions) while group g computes on `stream`.  The two device buffer pairs
        alternate ACROSS calls too, so back-to-back calls overlap the next call's first
        input copy and the previous call's last output copy with compute.  Returns when
        the work is queued.  sync_out=True: completion (output copies included) is ordered
        before later work on `stream`; False: returns the events of the last output
        copies instead (wait on them before reading out_host)."""
        import torch
        G = self.cfg.batch
        n = x_host.shape[0]
        if n % G or out_host.shape[0] != n:
            raise ValueError("forward_host: sample count must be a multiple of the context batch")
        if not (x_host.is_pinned() and out_host.is_pinned()):
            raise ValueError("forward_host: host buffers must be pinned")
        comp = torch.cuda.current_stream(self.device) if stream is None else stream
        if not hasattr(self, "_host_bufs"):
            xs = tuple(torch.empty((G,) + tuple(x_host.shape[1:]), dtype=torch.float32, device=self.device)
                       for _ in range(2))
            os_ = tuple(torch.empty((G,) + tuple(out_host.shape[1:]), dtype=torch.float32, device=self.device)
                        for _ in range(2))
            self._host_bufs = (xs, os_, self.tile_out_buffer(),
                               torch.cuda.Stream(self.device), torch.cuda.Stream(self.device))
            # per buffer: the last compute that read xs[b] / wrote os_[b], the last copy out of os_[b]
            self._host_state = {"comp_done": [None, None], "out_done": [None, None], "next": 0}
        xs, os_, tile_out, s_in, s_out = self._host_bufs
        stt = self._host_state
        for g in range(n // G):
            b = stt["next"]
            stt["next"] ^= 1
            sl = slice(g * G, (g + 1) * G)
            in_done = torch.cuda.Event()
            with torch.cuda.stream(s_in):
                if stt["comp_done"][b] is not None:   # the compute that read xs[b] is done
                    s_in.wait_event(stt["comp_done"][b])
                xs[b].copy_(x_host[sl], non_blocking=True)
                in_done.record(s_in)
            comp.wait_event(in_done)
            if stt["out_done"][b] is not None:        # os_[b] has been copied out
                comp.wait_event(stt["out_done"][b])
            self.forward(packed, xs[b], out=os_[b], tile_out=tile_out, stream=comp)
            cd = torch.cuda.Event()
            cd.record(comp)
            stt["comp_done"][b] = cd
            with torch.cuda.stream(s_out):
                s_out.wait_event(cd)
                out_host[sl].copy_(os_[b], non_blocking=True)
                od = torch.cuda.Event()
                od.record(s_out)
            stt["out_done"][b] = od
        last = [e for e in stt["out_done"] if e is not None]
        if sync_out:
            for e in last:
                comp.wait_event(e)
            return out_host
        return last

    # -- training step (include/orbit2.h "Training step") ----
    def train_info(self) -> orbit2_train_info:
        ti = orbit2_train_info()
        _check(lib.orbit2_train_plan(self.handle, C.byref(ti)), "orbit2_train_plan")
        return ti

    def train_bind(self, stream=None):
        """Allocate and bind the training workspace (activations kept for the backward)."""
        import torch
        ti = self.train_info()
        self.train_workspace = torch.empty(max(ti.workspace_bytes, 16), dtype=torch.uint8, device=self.device)
        with _on_device(self.device):
            _check(lib.orbit2_train_bind(self.handle, _ptr(self.train_workspace), ti.workspace_bytes,
                                         _stream(stream)), "orbit2_train_bind")
        self.tinfo = ti
        return ti

    def train_prepare(self, canonical_dev, stream=None):
        import torch
        _req(canonical_dev, torch.float32, "canonical_dev")
        with _on_device(self.device):
            _check(lib.orbit2_train_prepare(self.handle, _ptr(canonical_dev), _stream(stream)),
                   "orbit2_train_prepare")

    def train_forward(self, packed, x_dev, tile_out, stream=None):
        import torch
        _req(x_dev, torch.float32, "x_dev")
        _req(tile_out, torch.bfloat16, "tile_out")
        with _on_device(self.device):
            _check(lib.orbit2_train_forward(self.handle, _ptr(packed), _ptr(x_dev), _ptr(tile_out), _stream(stream)),
                   "orbit2_train_forward")

    def loss(self, out, truth, lam, delta, geo, loss_dev, dout, stream=None):
        import torch
        _req(out, torch.float32, "out")
        _req(truth, torch.float32, "truth")
        _req(loss_dev, torch.float64, "loss_dev")
        _req(dout, torch.float32, "dout")
        with _on_device(self.device):
            _check(lib.orbit2_loss(self.handle, _ptr(out), _ptr(truth), float(lam), float(delta), 1 if geo else 0,
                                   _ptr(loss_dev), _ptr(dout), _stream(stream)), "orbit2_loss")

    def train_backward(self, packed, dout, grad, stream=None):
        import torch
        _req(dout, torch.float32, "dout")
        _req(grad, torch.float32, "grad")
        with _on_device(self.device):
            _check(lib.orbit2_train_backward(self.handle, _ptr(packed), _ptr(dout), _ptr(grad), _stream(stream)),
                   "orbit2_train_backward")

    def train_step(self, packed, x_dev, truth, lam=1e-3, delta=1e-3, geo=True, bufs=None, stream=None):
        """One training step's forward, loss and backward over every rank-local tile:
        returns (loss per sample [B] float64, grad [canonical count] fp32, out).  The
        once-per-batch gradient all-reduce and the weight update are the caller's."""
        import torch
        cfg = self.cfg
        if bufs is None:
            bufs = self.train_buffers()
        tile_out, out, dout, loss_dev, grad = bufs
        self.train_forward(packed, x_dev, tile_out, stream)
        self.orbit2_stitch(tile_out, x_dev, 0, self.info.n_local_tiles, out, stream)
        self.loss(out, truth, lam, delta, geo, loss_dev, dout, stream)
        self.train_backward(packed, dout, grad, stream)
        return loss_dev, grad, out

    def train_buffers(self):
        import torch
        cfg = self.cfg
        tile_out = self.rank_tile_out()
        out = torch.empty((cfg.batch, cfg.K, self.sH, self.sW), dtype=torch.float32, device=self.device)
        dout = torch.empty_like(out)
        loss_dev = torch.empty(cfg.batch, dtype=torch.float64, device=self.device)
        grad = torch.empty(self.info.canonical_weight_count, dtype=torch.float32, device=self.device)
        return tile_out, out, dout, loss_dev, grad

    # -- the forward on compressed tokens (R41; include/orbit2.h) -------------------
    def compressed_forward(self, packed, x_dev, e_scale, max_side=8, threshold=0.1, sigma=1.0, low_frac=0.1,
                           high_frac=0.2, out=None, stream=None):
        """-> (out [B, K, sH, sW], leaves [n, 4] (image b T + t, u0, w0, side; patches of the tile's
        padded rectangle), n).  Every rank-local tile compressed on its own (R41, R42)."""
        import torch
        _req(x_dev, torch.float32, "x_dev")
        _req(e_scale, torch.float32, "e_scale")
        cp = orbit2_compression(max_side, threshold, sigma, low_frac, high_frac)
        ws, lv = C.c_int64(), C.c_int32()
        _check(lib.orbit2_compressed_plan(self.handle, C.byref(cp), C.byref(ws), C.byref(lv)),
               "orbit2_compressed_plan")
        if e_scale.shape[0] < lv.value:
            raise ValueError(f"e_scale needs {lv.value} rows")
        if getattr(self, "_cws", None) is None or self._cws.numel() < ws.value:
            self._cws = torch.empty(max(ws.value, 16), dtype=torch.uint8, device=self.device)
        cfg = self.cfg
        cap = cfg.batch * self.info.local_tokens
        leaves = torch.empty((max(cap, 1), 4), dtype=torch.int32, device=self.device)
        tile_out = self.tile_out_buffer()
        if out is None:
            out = torch.empty((cfg.batch, cfg.K, self.sH, self.sW), dtype=torch.float32, device=self.device)
        n = C.c_int32()
        with _on_device(self.device):
            _check(lib.orbit2_compressed_forward(self.handle, _ptr(packed), _ptr(x_dev), C.byref(cp), _ptr(e_scale),
                                                 _ptr(self._cws), self._cws.numel(), _ptr(tile_out), _ptr(leaves),
                                                 C.byref(n), _stream(stream)), "orbit2_compressed_forward")
        self.orbit2_stitch(tile_out, x_dev, 0, self.info.n_local_tiles, out, stream)
        return out, leaves[:n.value], n.value

    # -- CUDA-graph capture of the forward ----------------------
    def capture_forward(self, packed, x_dev, out, tile_out=None, stream=None):
        """Capture forward(packed, x_dev, out) -- every launch of the pass, on one stream, no
        host synchronisation inside -- into a CUDA graph; returns the graph (call .replay()).
        The buffers are baked in: refill x_dev in place between replays."""
        import torch
        if tile_out is None:
            tile_out = self.tile_out_buffer()
        self._graph_bufs = (packed, x_dev, out, tile_out)
        s = torch.cuda.Stream(self.device) if stream is None else stream
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.forward(packed, x_dev, out=out, tile_out=tile_out, stream=s)   # warm-up: attributes, tmaps
        torch.cuda.current_stream(self.device).wait_stream(s)
        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            self.forward(packed, x_dev, out=out, tile_out=tile_out, stream=s)
        return g

    # -- instrumentation ------------------------------------------------------
    def launch_count(self) -> int:
        return int(lib.orbit2_launch_count(self.handle))

    def set_profiling(self, on: bool):
        _check(lib.orbit2_set_profiling(self.handle, 1 if on else 0), "orbit2_set_profiling")

    def kernel_times(self) -> dict:
        n = lib.orbit2_kernel_times(self.handle, None, None, None, 0)
        names = (C.c_char_p * n)()
        launches = (C.c_int64 * n)()
        ms = (C.c_double * n)()
        lib.orbit2_kernel_times(self.handle, names, launches, ms, n)
        return {names[i].decode(): (int(launches[i]), float(ms[i])) for i in range(n)}


def adamw_step(w, grad, m, v, step, lr, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, stream=None):
    """orbit2_adamw_step on fp32 CUDA tensors of one size (in place: w, m, v)."""
    import torch
    for t, name in ((w, "w"), (grad, "grad"), (m, "m"), (v, "v")):
        _req(t, torch.float32, name)
    n = w.numel()
    if not (grad.numel() == m.numel() == v.numel() == n):
        raise ValueError("adamw_step: sizes differ")
    _check(lib.orbit2_adamw_step(_ptr(w), _ptr(grad), _ptr(m), _ptr(v), n, step, lr, beta1, beta2, eps, weight_decay,
                                 _stream(stream)), "orbit2_adamw_step")


class Compressor:
    """Adaptive spatial compression (include/orbit2.h): Canny +
    quad-tree partition of B fields, variable-size tokens and their decompression."""

    def __init__(self, *, batch, H, W, C, min_side, max_side, embed, threshold=0.05, sigma=1.0, low_frac=0.1,
                 high_frac=0.2, device=None):
        import torch
        self.cfg = orbit2_compress_config(batch, H, W, C, min_side, max_side, embed, threshold, sigma, low_frac,
                                          high_frac)
        ws, mp = _ct.c_int64(), _ct.c_int64()
        _check(lib.orbit2_compress_plan(_ct.byref(self.cfg), _ct.byref(ws), _ct.byref(mp)), "orbit2_compress_plan")
        self.device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        self.workspace = torch.empty(max(ws.value, 16), dtype=torch.uint8, device=self.device)
        self.max_patches = mp.value
        self.patches = torch.empty((max(mp.value, 1), 4), dtype=torch.int32, device=self.device)
        self.offsets = torch.empty(batch + 1, dtype=torch.int32, device=self.device)

    def partition(self, image_dev, edges=False, stream=None):
        """-> (patches [n, 4] int32 (image, row, col, side), offsets [B + 1], n, edge map or None)"""
        import torch
        _req(image_dev, torch.float32, "image_dev")
        e = torch.empty(image_dev.shape, dtype=torch.uint8, device=self.device) if edges else None
        n = _ct.c_int32()
        with _on_device(self.device):
            _check(lib.orbit2_compress_partition(_ct.byref(self.cfg), _ptr(image_dev), _ptr(self.workspace),
                                                 self.workspace.numel(), _ptr(e) if e is not None else None,
                                                 _ptr(self.patches), _ptr(self.offsets), _ct.byref(n), _stream(stream)),
                   "orbit2_compress_partition")
        return self.patches[:n.value], self.offsets, n.value, e

    def tokenize(self, feat_dev, patches, n, w_tok, b_tok, e_scale, stream=None):
        import torch
        for t, name in ((feat_dev, "feat_dev"), (w_tok, "w_tok"), (b_tok, "b_tok"), (e_scale, "e_scale")):
            _req(t, torch.float32, name)
        tok = torch.empty((max(n, 1), self.cfg.embed), dtype=torch.float32, device=self.device)
        with _on_device(self.device):
            _check(lib.orbit2_compress_tokenize(_ct.byref(self.cfg), _ptr(self.workspace), self.workspace.numel(),
                                                _ptr(feat_dev), _ptr(patches), n, _ptr(w_tok),
                                                _ptr(b_tok), _ptr(e_scale), _ptr(tok), _stream(stream)),
                   "orbit2_compress_tokenize")
        return tok[:n]

    def detokenize(self, tokens, patches, n, w_dec, b_dec, w_sm, b_sm, stream=None):
        import torch
        cf = self.cfg
        out = torch.empty((cf.batch, cf.C, cf.H, cf.W), dtype=torch.float32, device=self.device)
        work = torch.empty_like(out)
        with _on_device(self.device):
            _check(lib.orbit2_compress_detokenize(_ct.byref(cf), _ptr(self.workspace), self.workspace.numel(),
                                                  _ptr(tokens), _ptr(patches), n, _ptr(w_dec),
                                                  _ptr(b_dec), _ptr(w_sm), _ptr(b_sm), _ptr(work), _ptr(out),
                                                  _stream(stream)), "orbit2_compress_detokenize")
        return out
