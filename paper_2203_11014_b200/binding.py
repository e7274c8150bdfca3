"""Thin ctypes binding of libdhen.so (include/dhen.h).  Argument marshalling
only: every step of the DHEN path runs in the library's CUDA kernels; torch
provides device memory, streams and process groups.  There is no fallback: if
the library (or a GPU) is missing, calls raise."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libdhen.so")
WD_LIB_PATH = os.path.join(HERE, "libdhen_wd.so")   # debug build: bounded mbarrier waits (build.py --watchdog)

DOT, ATTN, CONV, DCN, LINEAR, MLP, DCN_LIT, DCN_FULL = range(8)
KIND_IDS = {"dot": DOT, "attn": ATTN, "conv": CONV, "dcn": DCN, "linear": LINEAR, "mlp": MLP, "dcn_lit": DCN_LIT,
            "dcn_full": DCN_FULL}
FP32, BF16 = 0, 1

STATUS = {0: "OK", 1: "E_CONFIG", 2: "E_SHAPE", 3: "E_ALIGN", 4: "E_STATE", 5: "E_CUDA", 6: "E_NCCL",
          7: "E_NONFINITE", 8: "E_NOMEM"}

# every symbol include/dhen.h and include/dhen_debug.h declare
EXPORTS = ("dhen_validate", "dhen_sizes", "dhen_group_numel", "dhen_nccl_id", "dhen_loopback_id", "dhen_comm_bytes",
           "dhen_init", "dhen_layer_fwd",
           "dhen_layer_bwd", "dhen_train_step", "dhen_train_step_graphed", "dhen_train_step_host", "dhen_forward", "dhen_zero_grad", "dhen_params_io",
           "dhen_grads_get", "dhen_launch_count", "dhen_last_error", "dhen_destroy", "dhen_profile",
           "dhen_profile_read", "dhen_debug_gemm", "dhen_debug_gemm_epi", "dhen_debug_last_gemm_tc",
           "dhen_debug_gemm_trace", "dhen_tuning_default", "dhen_set_tuning", "dhen_get_tuning",
           "dhen_debug_profile_trace", "dhen_fp_init", "dhen_fp_forward", "dhen_fp_backward_sgd", "dhen_fp_params_io",
           "dhen_fp_param_numel", "dhen_fp_bad_ids", "dhen_fp_destroy", "dhen_fp_init_dist", "dhen_fp_owned_tables",
           "dhen_fp_shard_plan")


class dhen_module(C.Structure):
    _fields_ = [("kind", C.c_int), ("l", C.c_int), ("heads", C.c_int), ("ffn_mult", C.c_int),
                ("conv_channels", C.c_int), ("conv_k", C.c_int), ("mlp_hidden", C.c_int * 2)]


class dhen_layer(C.Structure):
    _fields_ = [("n_modules", C.c_int), ("modules", C.POINTER(dhen_module)), ("ensemble", C.c_int),
                ("dense_in", C.c_int)]


ENSEMBLES = {"concat": 0, "sum": 1, "wsum": 2}   # dhen_ensemble


class dhen_config(C.Structure):
    _fields_ = [("m0", C.c_int), ("d", C.c_int), ("n_layers", C.c_int), ("layers", C.POINTER(dhen_layer)),
                ("dtype", C.c_int), ("ln_eps", C.c_float), ("batch_max_local", C.c_int),
                ("seed", C.c_ulonglong), ("optimizer", C.c_int), ("adam_beta1", C.c_float),
                ("adam_beta2", C.c_float), ("adam_eps", C.c_float), ("dense_tokens", C.c_int), ("recompute", C.c_int)]


class dhen_dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("world", C.c_int), ("nccl_id", C.c_ubyte * 128), ("fsdp", C.c_int),
                ("backend", C.c_int), ("grad_bf16", C.c_int)]


NCCL, LOOPBACK = 0, 1   # dhen_dist.backend


class dhen_op_stat(C.Structure):
    _fields_ = [("name", C.c_char * 40), ("launches", C.c_ulonglong), ("ms", C.c_double), ("flops", C.c_double),
                ("bytes", C.c_double), ("tc_launches", C.c_ulonglong)]


class dhen_tuning(C.Structure):
    """Schedule / fusion switches of one context (include/dhen_debug.h); defaults = measured best."""
    _fields_ = [(n, C.c_int) for n in ("overlap", "defer_join", "ln_fuse", "first_writer", "relu_bits", "fuse_db",
                                         "vdy", "trail", "bd_pre", "sym", "tstore", "pair", "pair_k", "attn_fused",
                                         "pdl", "gemm_simt", "dcn_fused", "dcn_tma", "ln_tma", "bn_max",
                                         "l2_prefetch", "wres", "resid_tma")]


class dhen_fp_config(C.Structure):
    """Feature processing layer (include/dhen.h, NEXT#4)."""
    _fields_ = [("n_sparse", C.c_int), ("rows", C.POINTER(C.c_longlong)), ("n_dense", C.c_int),
                ("n_hidden", C.c_int), ("hidden", C.POINTER(C.c_int)), ("n_dtok", C.c_int), ("d", C.c_int),
                ("dtype", C.c_int), ("max_batch", C.c_int), ("max_nnz", C.c_longlong), ("seed", C.c_ulonglong)]


class DhenError(RuntimeError):
    def __init__(self, call, status, msg):
        super().__init__(f"{call} -> DHEN_{STATUS.get(status, status)}: {msg}")
        self.status = status


_lib = None


def load(path: str = LIB_PATH):
    """Load libdhen.so (build it first with paper_2203_11014_b200.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise FileNotFoundError(f"{path} missing: run `python -m paper_2203_11014_b200.build`")
    lib = C.CDLL(path)
    vp, i, sz = C.c_void_p, C.c_int, C.c_size_t
    sig = {
        "dhen_validate": [C.POINTER(dhen_config)],
        "dhen_sizes": [C.POINTER(dhen_config), C.POINTER(dhen_dist), C.POINTER(sz), C.POINTER(sz)],
        "dhen_group_numel": [C.POINTER(dhen_config), C.POINTER(dhen_dist), i, C.POINTER(sz), C.POINTER(sz)],
        "dhen_nccl_id": [C.POINTER(C.c_ubyte)],
        "dhen_loopback_id": [C.POINTER(C.c_ubyte)],
        "dhen_init": [C.POINTER(dhen_config), C.POINTER(dhen_dist), vp, sz, vp, sz, vp, C.POINTER(vp)],
        "dhen_layer_fwd": [vp, i, vp, vp, i, vp],
        "dhen_layer_bwd": [vp, i, vp, vp, i, vp],
        "dhen_train_step": [vp, vp, vp, i, i, C.c_float, vp, vp, vp],
        "dhen_train_step_graphed": [vp, vp, vp, i, i, C.c_float, vp, vp, vp],
        "dhen_train_step_host": [vp, vp, vp, i, i, C.c_float, vp, i, vp],
        "dhen_forward": [vp, vp, i, vp, vp],
        "dhen_zero_grad": [vp, vp],
        "dhen_params_io": [vp, i, vp, i, vp],
        "dhen_grads_get": [vp, i, vp, vp],
        "dhen_profile": [vp, i],
        "dhen_profile_read": [vp, C.POINTER(dhen_op_stat), i, C.POINTER(i)],
        "dhen_debug_gemm": [C.POINTER(C.c_longlong), vp, vp, vp, i, i, i, vp, sz, vp],
        "dhen_debug_gemm_epi": [C.POINTER(C.c_longlong), vp, vp, vp, i, i, i, vp, sz, i, vp, vp, vp, vp],
        "dhen_set_tuning": [vp, C.POINTER(dhen_tuning)],
        "dhen_get_tuning": [vp, C.POINTER(dhen_tuning)],
        "dhen_debug_profile_trace": [vp, C.c_char_p],
        "dhen_fp_init": [C.POINTER(dhen_fp_config), vp, C.POINTER(vp)],
        "dhen_fp_forward": [vp, vp, vp, C.c_longlong, vp, i, vp, vp],
        "dhen_fp_backward_sgd": [vp, vp, C.c_float, vp],
        "dhen_fp_params_io": [vp, i, vp, i, vp],
        "dhen_fp_init_dist": [C.POINTER(dhen_fp_config), C.POINTER(dhen_dist), vp, C.POINTER(vp)],
        "dhen_fp_shard_plan": [C.POINTER(dhen_fp_config), i, C.POINTER(i), C.POINTER(i)],
    }
    for name, args in sig.items():
        f = getattr(lib, name, None)
        if f is None:   # (an older library build loaded for an A/B experiment; test_abi checks the exports)
            continue
        f.argtypes = args
        f.restype = C.c_int
    lib.dhen_last_error.restype = C.c_char_p
    lib.dhen_last_error.argtypes = []
    lib.dhen_launch_count.restype = C.c_ulonglong
    lib.dhen_launch_count.argtypes = [vp]
    if hasattr(lib, "dhen_comm_bytes"):
        lib.dhen_comm_bytes.restype = C.c_ulonglong
        lib.dhen_comm_bytes.argtypes = [vp]
    lib.dhen_debug_gemm_trace.restype = None
    lib.dhen_debug_gemm_trace.argtypes = [vp]
    lib.dhen_debug_last_gemm_tc.restype = C.c_int
    lib.dhen_debug_last_gemm_tc.argtypes = []
    if hasattr(lib, "dhen_tuning_default"):
        lib.dhen_tuning_default.restype = None
        lib.dhen_tuning_default.argtypes = [C.POINTER(dhen_tuning)]
    lib.dhen_destroy.restype = None
    lib.dhen_destroy.argtypes = [vp]
    if hasattr(lib, "dhen_fp_init"):
        lib.dhen_fp_param_numel.restype = C.c_longlong
        lib.dhen_fp_param_numel.argtypes = [C.POINTER(dhen_fp_config), i]
        lib.dhen_fp_bad_ids.restype = C.c_longlong
        lib.dhen_fp_bad_ids.argtypes = [vp]
        lib.dhen_fp_destroy.restype = None
        lib.dhen_fp_destroy.argtypes = [vp]
        lib.dhen_fp_owned_tables.restype = C.c_int
        lib.dhen_fp_owned_tables.argtypes = [vp, C.POINTER(C.c_int)]
    _lib = lib
    return lib


def _check(call, st):
    if st != 0:
        raise DhenError(call, st, load().dhen_last_error().decode())


@dataclass
class Module:
    kind: str
    l: int
    heads: int = 2
    ffn_mult: int = 4
    conv_channels: int = 4
    conv_k: int = 3
    mlp_hidden: Sequence[int] = (1024, 1024)


@dataclass
class Config:
    m0: int
    d: int
    layers: List[List[Module]]
    dtype: str = "bf16"
    batch_max_local: int = 1
    ln_eps: float = 1e-5
    seed: int = 0
    optimizer: str = "sgd"            # "sgd" (R18) | "adam" | "adam_bf16" (bf16 moments, R35)
    ensembles: Optional[Sequence[str]] = None   # per layer: "concat" (default) | "sum" | "wsum"
    recompute: int = 0                # bit 1: attention FFN hidden recomputed in the backward (NEXT#2)
    dense_tokens: int = 0             # R38: X0[:, :dense_tokens] injected into the dense_in layers
    dense_in: Optional[Sequence[bool]] = None   # per layer (NEXT#3)
    adam: Sequence[float] = (0.9, 0.999, 1e-8)
    _keep: list = field(default_factory=list, repr=False)

    def to_c(self) -> dhen_config:
        layers = (dhen_layer * len(self.layers))()
        keep = [layers]
        for n, L in enumerate(self.layers):
            mods = (dhen_module * len(L))()
            for i, s in enumerate(L):
                mods[i].kind = KIND_IDS[s.kind]
                mods[i].l = s.l
                mods[i].heads = s.heads
                mods[i].ffn_mult = s.ffn_mult
                mods[i].conv_channels = s.conv_channels
                mods[i].conv_k = s.conv_k
                mods[i].mlp_hidden[0] = s.mlp_hidden[0]
                mods[i].mlp_hidden[1] = s.mlp_hidden[1]
            layers[n].n_modules = len(L)
            layers[n].modules = C.cast(mods, C.POINTER(dhen_module))
            layers[n].ensemble = ENSEMBLES[self.ensembles[n]] if self.ensembles else 0
            layers[n].dense_in = int(bool(self.dense_in[n])) if self.dense_in else 0
            keep.append(mods)
        self._keep = keep
        return dhen_config(self.m0, self.d, len(self.layers), C.cast(layers, C.POINTER(dhen_layer)),
                           BF16 if self.dtype == "bf16" else FP32, self.ln_eps, self.batch_max_local, self.seed,
                           {"sgd": 0, "adam": 1, "adam_bf16": 2}[self.optimizer], *[float(x) for x in self.adam],
                           int(self.dense_tokens), int(self.recompute))

    def dims(self):
        out, m = [], self.m0
        for n, L in enumerate(self.layers):
            mo = sum(s.l for s in L) if not self.ensembles or self.ensembles[n] == "concat" else L[0].l
            out.append((m, mo))
            m = mo
        return out


def make_dist(rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None, fsdp: bool = True,
              backend: int = NCCL, grad_bf16: bool = False) -> dhen_dist:
    d = dhen_dist()
    d.rank, d.world, d.fsdp, d.backend, d.grad_bf16 = rank, world, int(fsdp), int(backend), int(grad_bf16)
    if nccl_id is not None:
        for k in range(128):
            d.nccl_id[k] = nccl_id[k]
    return d


def validate(cfg: Config) -> None:
    c = cfg.to_c()
    _check("dhen_validate", load().dhen_validate(C.byref(c)))


def sizes(cfg: Config, dist: Optional[dhen_dist] = None):
    c = cfg.to_c()
    s, w = C.c_size_t(), C.c_size_t()
    _check("dhen_sizes", load().dhen_sizes(C.byref(c), C.byref(dist or make_dist()), C.byref(s), C.byref(w)))
    return s.value, w.value


def group_numel(cfg: Config, group: int, dist: Optional[dhen_dist] = None):
    c = cfg.to_c()
    n, sh = C.c_size_t(), C.c_size_t()
    _check("dhen_group_numel", load().dhen_group_numel(C.byref(c), C.byref(dist or make_dist()), group,
                                                       C.byref(n), C.byref(sh)))
    return n.value, sh.value


def nccl_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check("dhen_nccl_id", load().dhen_nccl_id(buf))
    return bytes(buf)


def loopback_id() -> bytes:
    """A fresh id for a loopback group (backend=LOOPBACK): `world` virtual ranks in this process."""
    buf = (C.c_ubyte * 128)()
    _check("dhen_loopback_id", load().dhen_loopback_id(buf))
    return bytes(buf)


def debug_gemm(q, A, B, Cm, path=0, ws=None, stream=None):
    """Test hook: one contraction through the library's GEMM dispatcher (see dhen.h).
    Returns 0 (SIMT), 1 (tcgen05) or 2 (tcgen05 with CTA pairs); path 3 / 4 force pairs on / off."""
    import torch
    q = list(q) + [0] * (30 - len(q))
    arr = (C.c_longlong * 30)(*[int(v) for v in q])
    for t_ in (A, B, Cm):
        if t_.dtype not in (torch.bfloat16, torch.float32):
            raise TypeError(f"debug_gemm: unsupported dtype {t_.dtype}")
    abt = BF16 if A.dtype == torch.bfloat16 else FP32
    ct = BF16 if Cm.dtype == torch.bfloat16 else FP32
    if ws is None:
        ws = torch.empty(64 << 20, dtype=torch.uint8, device=A.device)
    s = stream if stream is not None else torch.cuda.current_stream()
    _check("dhen_debug_gemm", load().dhen_debug_gemm(arr, C.c_void_p(A.data_ptr()), C.c_void_p(B.data_ptr()),
                                                     C.c_void_p(Cm.data_ptr()), abt, ct, path,
                                                     C.c_void_p(ws.data_ptr()), ws.numel(), C.c_void_p(s.cuda_stream)))
    return int(load().dhen_debug_last_gemm_tc())


def tuning_default() -> dict:
    """The default (measured-best) schedule / fusion switches as a dict."""
    t = dhen_tuning()
    load().dhen_tuning_default(C.byref(t))
    return {n: getattr(t, n) for n, _ in dhen_tuning._fields_}


def debug_gemm_epi(q, A, B, Cm, mode, E=None, bias=None, aux=None, path=0, ws=None, stream=None):
    """Test hook: contraction + one fused epilogue (see dhen_debug_gemm_epi).  Returns True if tcgen05."""
    import torch
    q = list(q) + [0] * (30 - len(q))
    arr = (C.c_longlong * 30)(*[int(v) for v in q])
    abt = BF16 if A.dtype == torch.bfloat16 else FP32
    ct = BF16 if Cm.dtype == torch.bfloat16 else FP32
    if ws is None:
        ws = torch.empty(64 << 20, dtype=torch.uint8, device=A.device)
    s = stream if stream is not None else torch.cuda.current_stream()
    vp = lambda t: None if t is None else C.c_void_p(t.data_ptr())  # noqa: E731
    _check("dhen_debug_gemm_epi", load().dhen_debug_gemm_epi(arr, vp(A), vp(B), vp(Cm), abt, ct, path, vp(ws),
                                                             ws.numel(), mode, vp(E), vp(bias), vp(aux),
                                                             C.c_void_p(s.cuda_stream)))
    return int(load().dhen_debug_last_gemm_tc())


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class DHEN:
    """A DHEN stack bound to the current CUDA device.  State and work memory are
    torch uint8 CUDA tensors handed to the library (which carves them)."""

    def __init__(self, cfg: Config, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 fsdp: bool = True, stream=None, backend: int = NCCL, grad_bf16: bool = False):
        import torch
        self.torch = torch
        self.cfg = cfg
        self.lib = load()
        self.dist = make_dist(rank, world, nccl_id, fsdp, backend, grad_bf16)
        self._c = cfg.to_c()
        sb, wb = sizes(cfg, self.dist)
        dev = torch.device("cuda", torch.cuda.current_device())
        self.state = torch.empty(sb, dtype=torch.uint8, device=dev)
        self.work = torch.empty(wb, dtype=torch.uint8, device=dev)
        self.dtype = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
        ctx = C.c_void_p()
        _check("dhen_init", self.lib.dhen_init(C.byref(self._c), C.byref(self.dist), _ptr(self.state), sb,
                                               _ptr(self.work), wb, self._stream(stream), C.byref(ctx)))
        self.ctx = ctx
        self.n_groups = len(cfg.layers) + 1

    def _stream(self, stream=None):
        s = stream if stream is not None else self.torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)

    def close(self):
        if getattr(self, "ctx", None):
            self.lib.dhen_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def launches(self) -> int:
        return int(self.lib.dhen_launch_count(self.ctx))

    def comm_bytes(self) -> int:
        """Bytes this rank's collectives moved since init (dhen_comm_bytes)."""
        return int(self.lib.dhen_comm_bytes(self.ctx))

    def numel(self, group: int) -> int:
        return group_numel(self.cfg, group, self.dist)[0]

    def set_params(self, group: int, flat, stream=None):
        import numpy as np
        a = np.ascontiguousarray(flat, dtype=np.float32)
        assert a.size == self.numel(group), (a.size, self.numel(group))
        _check("dhen_params_io", self.lib.dhen_params_io(self.ctx, group, a.ctypes.data_as(C.c_void_p), 1,
                                                         self._stream(stream)))

    def get_params(self, group: int, stream=None):
        import numpy as np
        a = np.zeros(self.numel(group), np.float32)
        _check("dhen_params_io", self.lib.dhen_params_io(self.ctx, group, a.ctypes.data_as(C.c_void_p), 0,
                                                         self._stream(stream)))
        return a

    def get_grads(self, group: int, stream=None):
        import numpy as np
        a = np.zeros(self.numel(group), np.float32)
        _check("dhen_grads_get", self.lib.dhen_grads_get(self.ctx, group, a.ctypes.data_as(C.c_void_p),
                                                         self._stream(stream)))
        return a

    def zero_grad(self, stream=None):
        _check("dhen_zero_grad", self.lib.dhen_zero_grad(self.ctx, self._stream(stream)))

    def layer_fwd(self, n, x, y, stream=None):
        _check("dhen_layer_fwd", self.lib.dhen_layer_fwd(self.ctx, n, _ptr(x), _ptr(y), x.shape[0],
                                                         self._stream(stream)))

    def layer_bwd(self, n, dy, dx, stream=None):
        _check("dhen_layer_bwd", self.lib.dhen_layer_bwd(self.ctx, n, _ptr(dy), _ptr(dx), dy.shape[0],
                                                         self._stream(stream)))

    def train_step(self, x0, labels, lr, B_global=None, loss=None, dx0=None, stream=None):
        B = x0.shape[0]
        _check("dhen_train_step", self.lib.dhen_train_step(self.ctx, _ptr(x0), _ptr(labels), B,
                                                           B_global or B, float(lr), _ptr(loss), _ptr(dx0),
                                                           self._stream(stream)))

    def profile(self, enable, keep_overlap: bool = False):
        """Per-op CUDA-event timing on (serialised side stream, or concurrency kept) / off."""
        _check("dhen_profile", self.lib.dhen_profile(self.ctx, (2 if keep_overlap else 1) if enable else 0))

    def profile_trace(self, path: str):
        """Per-op timeline (tag, stream, start, end ms) of the last profiled pass -> CSV (tools/timeline.py)."""
        _check("dhen_debug_profile_trace", self.lib.dhen_debug_profile_trace(self.ctx, path.encode()))

    def tuning(self) -> dict:
        t = dhen_tuning()
        _check("dhen_get_tuning", self.lib.dhen_get_tuning(self.ctx, C.byref(t)))
        return {n: getattr(t, n) for n, _ in dhen_tuning._fields_}

    def set_tuning(self, **kw):
        """Change this context's schedule / fusion switches (dhen_debug.h dhen_tuning): set_tuning(overlap=0)."""
        t = dhen_tuning()
        _check("dhen_get_tuning", self.lib.dhen_get_tuning(self.ctx, C.byref(t)))
        for k, v in kw.items():
            if not hasattr(t, k):
                raise KeyError(k)
            setattr(t, k, int(v))
        _check("dhen_set_tuning", self.lib.dhen_set_tuning(self.ctx, C.byref(t)))

    def profile_read(self):
        """[{name, launches, ms, flops, bytes}] aggregated per op tag."""
        cap = 256
        arr = (dhen_op_stat * cap)()
        n = C.c_int()
        _check("dhen_profile_read", self.lib.dhen_profile_read(self.ctx, arr, cap, C.byref(n)))
        return [{"name": arr[k].name.decode(), "launches": arr[k].launches, "ms": arr[k].ms,
                 "flops": arr[k].flops, "bytes": arr[k].bytes,
                 "tc_launches": arr[k].tc_launches} for k in range(min(n.value, cap))]

    def train_step_graphed(self, x0, labels, lr, B_global=None, loss=None, dx0=None, stream=None):
        """train_step replayed from a CUDA graph (captured on the first call with these buffers)."""
        B = x0.shape[0]
        _check("dhen_train_step_graphed", self.lib.dhen_train_step_graphed(
            self.ctx, _ptr(x0), _ptr(labels), B, B_global or B, float(lr), _ptr(loss), _ptr(dx0),
            self._stream(stream)))

    def train_step_host(self, x0_host, labels_host, lr, B_global=None, loss_host=None, sync=True, stream=None):
        """One step from (pinned) host tensors through the C ABI's host-buffer entry: the library uploads them,
        runs the step and writes this rank's loss into loss_host (a 1-element host fp32 tensor)."""
        B = x0_host.shape[0]
        _check("dhen_train_step_host", self.lib.dhen_train_step_host(
            self.ctx, _ptr(x0_host), _ptr(labels_host), B, B_global or B, float(lr), _ptr(loss_host),
            1 if sync else 0, self._stream(stream)))

    def forward(self, x0, logits, stream=None):
        _check("dhen_forward", self.lib.dhen_forward(self.ctx, _ptr(x0), x0.shape[0], _ptr(logits),
                                                     self._stream(stream)))


class FeatureProcessing:
    """The feature processing layer in front of the stack (NEXT#4, include/dhen.h dhen_fp_*): sum-pooled
    embedding bags + bottom MLP -> X0 [B][n_dtok + n_sparse][d].  Argument marshalling only."""

    def __init__(self, rows, n_dense, hidden, n_dtok, d, dtype="bf16", max_batch=1, max_nnz=0, seed=0, stream=None,
                 rank=0, world=1, comm_id=None, backend=NCCL):
        import torch
        self.torch = torch
        self.lib = load()
        self.rows, self.n_dense, self.hidden, self.n_dtok, self.d = list(rows), n_dense, list(hidden), n_dtok, d
        self.dtype = torch.bfloat16 if dtype == "bf16" else torch.float32
        self._rows = (C.c_longlong * max(1, len(self.rows)))(*self.rows)
        self._hidden = (C.c_int * max(1, len(self.hidden)))(*self.hidden)
        self._c = dhen_fp_config(len(self.rows), self._rows, n_dense, len(self.hidden), self._hidden, n_dtok, d,
                                 BF16 if dtype == "bf16" else FP32, max_batch, max_nnz, seed)
        h = C.c_void_p()
        self.world, self.rank = world, rank
        if world > 1:   # column-sharded tables over `world` ranks (R36); comm_id from nccl_id() / loopback_id()
            self._dist = make_dist(rank, world, comm_id, True, backend)
            _check("dhen_fp_init_dist", self.lib.dhen_fp_init_dist(C.byref(self._c), C.byref(self._dist),
                                                                   self._stream(stream), C.byref(h)))
        else:
            _check("dhen_fp_init", self.lib.dhen_fp_init(C.byref(self._c), self._stream(stream), C.byref(h)))
        self.h = h
        self.m0 = n_dtok + len(self.rows)
        self.n_params = len(self.rows) + 2 * ((len(self.hidden) + 1) if n_dtok > 0 else 0)

    def _stream(self, stream=None):
        s = stream if stream is not None else self.torch.cuda.current_stream()
        return C.c_void_p(s.cuda_stream)

    def numel(self, which):
        return self.lib.dhen_fp_param_numel(C.byref(self._c), which)

    def owned_tables(self):
        n = self.lib.dhen_fp_owned_tables(self.h, None)
        out = (C.c_int * max(1, n))()
        self.lib.dhen_fp_owned_tables(self.h, out)
        return list(out)[:n]

    def plan(self, world):
        """(shards per table, owner rank of each shard) of the column-shard plan for `world` ranks."""
        S = (C.c_int * max(1, len(self.rows)))()
        own = (C.c_int * max(1, len(self.rows) * (self.d // 4)))()
        _check("dhen_fp_shard_plan", self.lib.dhen_fp_shard_plan(C.byref(self._c), world, S, own))
        S = list(S)[:len(self.rows)]
        return S, list(own)[:sum(S)]

    def forward(self, ids, offsets, dense, x0, stream=None):
        """ids / offsets int32 CUDA tensors (CSR bags, sample-major), dense [B][n_dense], x0 [B][m0][d] out."""
        B = x0.shape[0]
        _check("dhen_fp_forward", self.lib.dhen_fp_forward(self.h, _ptr(ids), _ptr(offsets), int(ids.numel()),
                                                           _ptr(dense), B, _ptr(x0), self._stream(stream)))
        self._fwd_refs = (ids, offsets, dense, x0)   # the library reads them again in backward_sgd

    def backward_sgd(self, dx0, lr, stream=None):
        _check("dhen_fp_backward_sgd", self.lib.dhen_fp_backward_sgd(self.h, _ptr(dx0), C.c_float(lr),
                                                                     self._stream(stream)))
        self._bwd_refs, self._fwd_refs = (dx0, getattr(self, "_fwd_refs", None)), None   # (until the next call)

    def get(self, which):
        import numpy as np
        out = np.zeros(self.numel(which), np.float32)   # (sharded tables: this rank's columns, zeros elsewhere)
        _check("dhen_fp_params_io", self.lib.dhen_fp_params_io(self.h, which, out.ctypes.data_as(C.c_void_p), 0,
                                                               self._stream()))
        return out

    def set(self, which, values):
        import numpy as np
        a = np.ascontiguousarray(values, np.float32).reshape(-1)
        assert a.size == self.numel(which)
        _check("dhen_fp_params_io", self.lib.dhen_fp_params_io(self.h, which, a.ctypes.data_as(C.c_void_p), 1,
                                                               self._stream()))

    def bad_ids(self):
        return self.lib.dhen_fp_bad_ids(self.h)

    def close(self):
        if getattr(self, "h", None):
            self.lib.dhen_fp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
