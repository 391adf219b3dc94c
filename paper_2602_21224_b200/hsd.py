"""Thin ctypes binding of include/hsd.h (argument marshalling only).

Every arithmetic step of the path runs in libhsd.so's CUDA kernels; this module
only converts Python values to the C structs/pointers and back. There is no
fallback: if libhsd.so is missing or cannot be loaded, `load()` raises.
Names follow the C ABI: init_model / prefill / build_tree / verify_tree /
accept_and_compact / step / destroy.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libhsd.so")

HSD_OK, HSD_EINVAL, HSD_ENOMEM, HSD_ECUDA, HSD_ENCCL, HSD_ESTATE, HSD_EUNSUP, HSD_EDEVICE = 0, -1, -2, -3, -4, -5, -6, -7
STATUS = {0: "OK", -1: "EINVAL", -2: "ENOMEM", -3: "ECUDA", -4: "ENCCL", -5: "ESTATE", -6: "EUNSUP", -7: "EDEVICE"}
FP32_VERIFY, BF16 = 0, 1
GREEDY, STOCHASTIC = 0, 1
FLAG_RESAMPLE, FLAG_FUSION, FLAG_PLANTED, FLAG_ZERO_TABLE, FLAG_TCGEN05, FLAG_TABLE_FP8 = 1, 2, 4, 8, 16, 32
FLAG_NO_FIRST_TOKEN = 1 << 6
FLAG_TOKEN_AR = 1 << 7
MAX_PLANT_DEPTH = 16
SHARD_NONE, SHARD_NCCL, SHARD_SIM = 0, 1, 2

EXPORTS = ["hsd_config_defaults", "hsd_init_model", "hsd_prefill", "hsd_set_plant", "hsd_set_block_table", "hsd_build_tree",
           "hsd_force_tree", "hsd_verify_tree", "hsd_accept_and_compact", "hsd_step", "hsd_step_host",
           "hsd_sync", "hsd_get_tensor", "hsd_kernel_launches", "hsd_destroy", "hsd_last_error",
           "hsd_profile", "hsd_profile_read", "hsd_debug_gemm", "hsd_nccl_unique_id", "hsd_admit", "hsd_kstamp", "hsd_kstamp_read", "hsd_kstamp_read_attention",
           "hsd_debug_gumbel"]
PROFILE_CATEGORIES = ["gemm_verify", "gemm_draft", "head_verify", "head_draft", "attn_verify", "attn_draft",
                      "tree", "resample", "walk", "compact", "rowwise"]


class HsdConfig(C.Structure):
    _fields_ = [(f, C.c_int32) for f in ("vocab", "hidden", "layers", "q_heads", "kv_heads", "head_dim", "ffn")] + \
        [("rope_theta", C.c_float), ("rms_eps", C.c_float)] + \
        [(f, C.c_int32) for f in ("steps_N", "branch_k", "budget_B", "resample_budget_Br", "resample_threshold_r",
                                   "hot_tokens", "table_rank", "max_batch", "max_ctx", "page_size", "precision",
                                   "accept_mode")] + \
        [("temperature", C.c_float), ("seed", C.c_uint64), ("flags", C.c_uint32), ("req_offset", C.c_int32),
         ("vocab_perm", C.POINTER(C.c_int32)), ("plant_rates", C.c_float * MAX_PLANT_DEPTH),
         ("vocab_shards", C.c_int32), ("shard_rank", C.c_int32), ("shard_mode", C.c_int32),
         ("nccl_id", C.c_uint8 * 128)]


class TreeView(C.Structure):
    _fields_ = [("tok", C.c_void_p), ("par", C.c_void_p), ("depth", C.c_void_p), ("logjoint", C.c_void_p),
                ("n", C.c_void_p), ("anc", C.c_void_p), ("batch", C.c_int32), ("t_max", C.c_int32),
                ("anc_words", C.c_int32)]


class VerifyView(C.Structure):
    _fields_ = [("logits", C.c_void_p), ("argmax", C.c_void_p), ("hidden", C.c_void_p), ("batch", C.c_int32),
                ("t_max", C.c_int32), ("vocab", C.c_int32), ("hidden_dim", C.c_int32)]


class Tensor(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("dtype", C.c_int32), ("ndim", C.c_int32), ("dims", C.c_int64 * 4)]


_lib = None


def load(path: str = LIB_PATH):
    """dlopen libhsd.so and declare signatures. Raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"{path} not built: run `python -m paper_2602_21224_b200.build` "
                           "(there is no CPU fallback)")
    lib = C.CDLL(path)
    P, I32, I64, VP = C.POINTER, C.c_int32, C.c_int64, C.c_void_p
    sig = {
        "hsd_config_defaults": (None, [P(HsdConfig)]),
        "hsd_init_model": (I32, [P(HsdConfig), C.c_int, VP, P(VP)]),
        "hsd_prefill": (I32, [VP, I32, P(I32), I32, P(I32), VP]),
        "hsd_set_plant": (I32, [VP, P(I32), I32]),
        "hsd_set_block_table": (I32, [VP, P(I32)]),
        "hsd_build_tree": (I32, [VP, P(TreeView)]),
        "hsd_force_tree": (I32, [VP, P(I32), P(I32), P(I32), P(I32)]),
        "hsd_verify_tree": (I32, [VP, P(VerifyView)]),
        "hsd_accept_and_compact": (I32, [VP, VP, VP]),
        "hsd_step": (I32, [VP, VP, VP]),
        "hsd_step_host": (I32, [VP, P(I32), P(I32)]),
        "hsd_sync": (I32, [VP]),
        "hsd_get_tensor": (I32, [VP, C.c_char_p, P(Tensor)]),
        "hsd_kernel_launches": (I64, [VP]),
        "hsd_destroy": (I32, [VP]),
        "hsd_last_error": (C.c_char_p, [VP]),
        "hsd_profile": (I32, [VP, C.c_int]),
        "hsd_debug_gemm": (I32, [VP, I32, VP, I32, VP, I32, I32, I32, I32, I32, I32, I32, VP]),
        "hsd_profile_read": (I32, [VP, C.c_char_p, P(C.c_double), P(I64), P(C.c_double), P(C.c_double)]),
        "hsd_nccl_unique_id": (I32, [P(C.c_uint8)]),
        "hsd_admit": (I32, [VP, I32, P(I32), I32, I32, VP]),
        "hsd_kstamp": (I32, [VP, C.c_int]),
        "hsd_kstamp_read": (I32, [VP, P(C.c_double), P(I64), P(C.c_double), P(C.c_double)]),
        "hsd_kstamp_read_attention": (I32, [VP, P(C.c_double), P(I64)]),
        "hsd_debug_gumbel": (I32, [VP, I32, I32, C.c_float, C.c_uint64, I32, I32, I32, VP, VP, VP, VP]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype, fn.argtypes = res, args
    _lib = lib
    return lib


class HsdError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def _i32(a):
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int32))


def make_config(model_cfg, *, precision=BF16, max_batch=None, max_ctx=None, seed=0, flags=None,
                accept=None, temperature=None, req_offset=0, vocab_perm=None, plant_rates=None,
                page_size=64, tcgen05=False, vocab_shards=1, shard_rank=0, shard_mode=SHARD_NONE, nccl_id=None):
    """Build an HsdConfig from a shape description (any object with the
    attributes of synth.Config). Returns (config, keepalive)."""
    lib = load()
    c = HsdConfig()
    lib.hsd_config_defaults(C.byref(c))
    for f in ("vocab", "hidden", "layers", "q_heads", "kv_heads", "head_dim", "ffn", "steps_N", "branch_k",
              "budget_B", "resample_budget_Br", "resample_threshold_r", "hot_tokens"):
        setattr(c, f, int(getattr(model_cfg, f)))
    c.rope_theta = float(model_cfg.rope_theta)
    c.rms_eps = float(model_cfg.rms_eps)
    c.table_rank = int(model_cfg.table_rank)
    c.max_batch = int(max_batch if max_batch is not None else model_cfg.batch)
    c.max_ctx = int(max_ctx if max_ctx is not None else model_cfg.prompt_len + model_cfg.max_new + 8)
    c.page_size = int(page_size)
    c.precision = int(precision)
    accept = accept if accept is not None else model_cfg.accept
    c.accept_mode = STOCHASTIC if accept in ("stochastic", STOCHASTIC) else GREEDY
    c.temperature = float(temperature if temperature is not None else model_cfg.temperature)
    c.seed = int(seed)
    c.flags = int(flags if flags is not None else (FLAG_RESAMPLE | FLAG_FUSION)) | (FLAG_TCGEN05 if tcgen05 else 0)
    c.req_offset = int(req_offset)
    c.vocab_shards, c.shard_rank, c.shard_mode = int(vocab_shards), int(shard_rank), int(shard_mode)
    if nccl_id is not None:
        b = bytes(nccl_id)
        if len(b) != 128:
            raise ValueError("nccl_id must be 128 bytes (hsd_nccl_unique_id)")
        C.memmove(c.nccl_id, b, 128)
    keep = []
    if vocab_perm is not None:
        arr, ptr = _i32(vocab_perm)
        keep.append(arr)
        c.vocab_perm = ptr
    if plant_rates is not None:
        for i, a in enumerate(list(plant_rates)[:MAX_PLANT_DEPTH]):
            c.plant_rates[i] = float(a)
    return c, keep


class _CAI:
    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class Context:
    """One hsd_ctx (one device, one stream, <= max_batch requests)."""

    def __init__(self, cfg: HsdConfig, device: int = 0, stream=None, keepalive=()):
        self.lib = load()
        self._keep = list(keepalive)
        self.cfg = cfg
        h = C.c_void_p()
        st = C.c_void_p(int(stream) if stream is not None else 0)
        s = self.lib.hsd_init_model(C.byref(cfg), device, st, C.byref(h))
        if s != HSD_OK:
            raise HsdError(s, "hsd_init_model failed (see stderr)")
        self.h = h
        self.device = device
        self.batch = 0

    def _check(self, s):
        if s != HSD_OK:
            raise HsdError(s, self.lib.hsd_last_error(self.h).decode())

    # --- the C ABI ------------------------------------------------------
    def prefill(self, tokens, lens=None, d_first=None):
        tokens = np.atleast_2d(np.asarray(tokens, dtype=np.int32))
        lens = np.full(tokens.shape[0], tokens.shape[1], np.int32) if lens is None else np.asarray(lens, np.int32)
        t, tp = _i32(tokens)
        l, lp = _i32(lens)
        self._check(self.lib.hsd_prefill(self.h, tokens.shape[0], tp, tokens.shape[1], lp,
                                         C.c_void_p(d_first or 0)))
        self.batch = tokens.shape[0]

    def admit(self, slot, tokens, req_id, d_first=None):
        """hsd_admit: a new (ragged-length) prompt into batch slot `slot`; the
        other slots keep decoding (continuous batching). `req_id` is the new
        request's global id for its random streams (must be fresh)."""
        t, tp = _i32(np.asarray(tokens, dtype=np.int32).ravel())
        self._check(self.lib.hsd_admit(self.h, int(slot), tp, t.size, int(req_id), C.c_void_p(d_first or 0)))

    def set_plant(self, plant):
        plant = np.atleast_2d(np.asarray(plant, dtype=np.int32))
        a, p = _i32(plant)
        self._check(self.lib.hsd_set_plant(self.h, p, plant.shape[1]))

    def set_block_table(self, table):
        """hsd_set_block_table: [max_batch, pages_per_req] page permutation (paged KV)."""
        t, tp = _i32(np.asarray(table, dtype=np.int32).ravel())
        self._check(self.lib.hsd_set_block_table(self.h, tp))

    def build_tree(self):
        v = TreeView()
        self._check(self.lib.hsd_build_tree(self.h, C.byref(v)))
        return v

    def force_tree(self, tok, par, depth, n):
        arrs = [_i32(x) for x in (tok, par, depth, n)]
        self._check(self.lib.hsd_force_tree(self.h, *[p for _, p in arrs]))

    def verify_tree(self):
        v = VerifyView()
        self._check(self.lib.hsd_verify_tree(self.h, C.byref(v)))
        return v

    def accept_and_compact(self, d_emitted=None, d_n=None):
        self._check(self.lib.hsd_accept_and_compact(self.h, C.c_void_p(d_emitted or 0), C.c_void_p(d_n or 0)))

    def step(self, d_emitted=None, d_n=None):
        self._check(self.lib.hsd_step(self.h, C.c_void_p(d_emitted or 0), C.c_void_p(d_n or 0)))

    def step_host(self):
        N = self.cfg.steps_N
        em = np.empty((self.batch, N + 1), np.int32)
        n = np.empty(self.batch, np.int32)
        self._check(self.lib.hsd_step_host(self.h, em.ctypes.data_as(C.POINTER(C.c_int32)),
                                           n.ctypes.data_as(C.POINTER(C.c_int32))))
        return em, n

    def sync(self):
        self._check(self.lib.hsd_sync(self.h))

    def profile(self, enable: bool):
        self._check(self.lib.hsd_profile(self.h, 1 if enable else 0))

    def profile_read(self):
        """{category: (ms, launches, algorithmic bytes, flops)}"""
        out = {}
        for cat in PROFILE_CATEGORIES:
            ms, n, by, fl = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
            self._check(self.lib.hsd_profile_read(self.h, cat.encode(), C.byref(ms), C.byref(n), C.byref(by),
                                                  C.byref(fl)))
            out[cat] = (ms.value, n.value, by.value, fl.value)
        return out

    def kstamp(self, enable: bool):
        self._check(self.lib.hsd_kstamp(self.h, 1 if enable else 0))

    def kstamp_read(self):
        """(avg us per stamped verify-GEMM launch, samples, bytes / launch, flops / launch)"""
        us, n, by, fl = C.c_double(), C.c_int64(), C.c_double(), C.c_double()
        self._check(self.lib.hsd_kstamp_read(self.h, C.byref(us), C.byref(n), C.byref(by), C.byref(fl)))
        return us.value, n.value, by.value, fl.value

    def kstamp_read_attention(self):
        """(avg us per stamped verify tree-attention launch incl. its split merge, samples)"""
        us, n = C.c_double(), C.c_int64()
        self._check(self.lib.hsd_kstamp_read_attention(self.h, C.byref(us), C.byref(n)))
        return us.value, n.value

    def kernel_launches(self) -> int:
        return int(self.lib.hsd_kernel_launches(self.h))

    def tensor(self, name, sync=True):
        """Zero-copy torch view of a named device tensor (hsd_get_tensor). By
        default the context stream is synchronised first, so the view is not read
        (e.g. by .cpu() on torch's current stream) while kernels still write it."""
        import torch
        if sync:
            self.sync()
        t = Tensor()
        self._check(self.lib.hsd_get_tensor(self.h, name.encode(), C.byref(t)))
        shape = [t.dims[i] for i in range(t.ndim)]
        typestr = {0: "<f4", 1: "<i2", 2: "<i4", 3: "<u8", 4: "|u1"}[t.dtype]
        x = torch.as_tensor(_CAI(t.ptr, shape, typestr), device=f"cuda:{self.device}")
        return x.view(torch.bfloat16) if t.dtype == 1 else x

    def destroy(self):
        if getattr(self, "h", None):
            self.lib.hsd_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def debug_gemm(A, W, C, accumulate=False, use_tc=False, stream=0):
    """C (+)= A @ W^T with the library's GEMM kernels (torch CUDA tensors;
    marshalling only). A, W: bf16 or fp32, row-major; C: fp32."""
    import torch
    lib = load()
    dtype = 1 if A.dtype == torch.bfloat16 else 0
    M, K = A.shape
    N = W.shape[0]
    s = lib.hsd_debug_gemm(A.data_ptr(), A.stride(0), W.data_ptr(),
                           W.stride(0), C.data_ptr(), C.stride(0), M, N, K, int(accumulate), dtype,
                           2 if use_tc == "swiglu" else int(bool(use_tc)), stream)
    if s != HSD_OK:
        raise HsdError(s, "hsd_debug_gemm")


def debug_gumbel(logits, rows, slots, temperature, seed, req, step, stream=0):
    """hsd_debug_gumbel: Gumbel-max draws (the walk's device code) for logits rows
    `rows` (torch CUDA fp32 [*, V]) with Philox slots `slots` (int32 CUDA tensors)."""
    import torch
    out = torch.empty(rows.numel(), dtype=torch.int32, device=logits.device)
    s = load().hsd_debug_gumbel(logits.data_ptr(), logits.stride(0), logits.shape[1], float(temperature), int(seed),
                                int(req), int(step), rows.numel(), rows.data_ptr(), slots.data_ptr(),
                                out.data_ptr(), stream)
    if s != HSD_OK:
        raise HsdError(s, "hsd_debug_gumbel")
    return out


def nccl_unique_id() -> bytes:
    """hsd_nccl_unique_id: 128 bytes on shard 0, to broadcast to the other shards."""
    buf = (C.c_uint8 * 128)()
    s = load().hsd_nccl_unique_id(buf)
    if s != HSD_OK:
        raise HsdError(s, "hsd_nccl_unique_id (libnccl.so.2 not loadable?)")
    return bytes(buf)


def shard_nccl_id(group=None) -> bytes:
    """Bootstrap of the vocab-shard NCCL group over an initialised
    torch.distributed process group (any backend): shard 0 creates the id
    (hsd_nccl_unique_id), every rank receives the same 128 bytes."""
    import torch.distributed as dist
    obj = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return obj[0]


def vocab_shard_bounds(V: int, G: int):
    """Column bounds lo_0..lo_G of the G vocab shards (include/hsd.h): lo_s =
    floor(s*V/G / 128) * 128, lo_G = V. Host-side mirror for tests/planning."""
    return [(s * V // G) // 128 * 128 for s in range(G)] + [V]


def init_model(model_cfg, device=0, stream=None, **kw) -> Context:
    cfg, keep = make_config(model_cfg, **kw)
    return Context(cfg, device=device, stream=stream, keepalive=keep)
