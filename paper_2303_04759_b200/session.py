"""Python binding of libtrainc_b200.so -- the b200 training-step runtime.

    s = Session(ModelConfig.bert_base(B=32))   # graph -> autodiff -> fusion -> VM
    s.init_params()
    ids, labels = synthetic_batch(s.cfg)
    s.set_batch(ids, labels); s.step(); loss = s.loss()

Every kernel the step launches is a libtcb200 sm_100a kernel; there is no CPU
path here (creating a session on a machine without a B200 raises).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field, fields

import numpy as np

from . import runtime

PKG = os.path.dirname(os.path.abspath(__file__))
HOST_LIB = os.path.join(PKG, "lib", "libtrainc_b200.so")

_lib = None


def lib():
    global _lib
    if _lib is None:
        runtime.lib()  # libtcb200 first (dependency, rpath $ORIGIN)
        if not os.path.exists(HOST_LIB):
            raise RuntimeError(f"{HOST_LIB} not built; run __graft_entry__.build()")
        L = ctypes.CDLL(HOST_LIB)
        L.tb_last_error.restype = ctypes.c_char_p
        L.tb_session_create.restype = ctypes.c_void_p
        L.tb_session_create.argtypes = [ctypes.c_char_p, ctypes.c_int]
        for f in ("tb_session_destroy", "tb_session_init_params", "tb_session_sync",
                  "tb_session_fetch_loss"):
            getattr(L, f).argtypes = [ctypes.c_void_p]
        L.tb_session_step.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.tb_session_info.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
        L.tb_session_set_batch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.tb_session_loss_value.restype = ctypes.c_float
        L.tb_session_loss_value.argtypes = [ctypes.c_void_p]
        L.tb_session_stream.restype = ctypes.c_void_p
        L.tb_session_stream.argtypes = [ctypes.c_void_p]
        L.tb_session_param.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.POINTER(ctypes.c_void_p),
                                       ctypes.POINTER(ctypes.c_int64)]
        L.tb_session_ids_buffer.restype = ctypes.c_void_p
        L.tb_session_ids_buffer.argtypes = [ctypes.c_void_p]
        L.tb_session_labels_buffer.restype = ctypes.c_void_p
        L.tb_session_labels_buffer.argtypes = [ctypes.c_void_p]
        L.tb_session_text.restype = ctypes.c_char_p
        L.tb_session_text.argtypes = [ctypes.c_void_p, ctypes.c_char_p]
        L.tb_session_segments.restype = ctypes.c_char_p
        L.tb_session_segments.argtypes = [ctypes.c_void_p]
        L.tb_session_set_comm.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.tb_graph_info.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
        L.tb_graph_text.restype = ctypes.c_char_p
        L.tb_graph_text.argtypes = [ctypes.c_char_p, ctypes.c_char_p]
        L.tb_synthetic_batch.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_void_p, ctypes.c_int]
        L.tb_cache_stats.argtypes = [ctypes.POINTER(ctypes.c_int64)]
        L.tb_cache_clear.argtypes = []
        L.tb_text_reprint.restype = ctypes.c_char_p
        L.tb_text_reprint.argtypes = [ctypes.c_char_p]
        L.tb_autocast_info.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_char_p,
                                       ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
        L.tb_tnsr_save.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(ctypes.c_int64)]
        L.tb_tnsr_header.argtypes = [ctypes.c_char_p, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                     ctypes.POINTER(ctypes.c_int64), ctypes.c_int]
        L.tb_tnsr_load.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int64]
        L.tb_session_save_param.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_char_p]
        L.tb_session_load_param.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_char_p]
        L.tb_session_profile.restype = ctypes.c_char_p
        L.tb_session_profile.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.tb_session_profile_inner.restype = ctypes.c_char_p
        L.tb_session_profile_inner.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
        L.tb_derive_priorities.restype = ctypes.c_char_p
        L.tb_derive_priorities.argtypes = [ctypes.c_char_p]
        L.tb_memsched_text.restype = ctypes.c_char_p
        L.tb_memsched_text.argtypes = [ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int64, ctypes.c_int]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise RuntimeError(lib().tb_last_error().decode())


@dataclass
class ModelConfig:
    """Mirrors tb::ModelCfg (host/models.hpp)."""
    kind: str = "bert"
    L: int = 2
    H: int = 128
    A: int = 2
    F: int = 512
    V: int = 1024
    S: int = 128
    B: int = 8
    dtype: str = "f32"
    p: float = 0.0
    opt: str = "sgd"
    lr: float = 0.01
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-6
    seed_w: int = 42
    seed_d: int = 1234
    seed_drop: int = 7
    world: int = 1
    fuse: int = 1
    bucket_mb: float = 25.0  # ZeRO gradient bucket (f32 MB; 0: one per parameter segment)
    zero: int = 0            # ZeRO data plane at world 1 (identity collectives, comm stream)
    rules: int = 1           # rule-based fusion of elementwise runs into ew_closure kernels
    disable_patterns: str = ""  # comma list of b200 FusionPattern names switched off
    flash: int = 1           # bf16 attention lse mode (P recomputed in the bwd): 1 for S > 128, 2 always, 0 never
    extra: dict = field(default_factory=dict)  # runtime keys: budget, schedule, rank

    def cfg_string(self, model_only: bool = False) -> str:
        kv = [f"{f.name}={getattr(self, f.name)}" for f in fields(self) if f.name != "extra"]
        if not model_only:
            kv += [f"{k}={v}" for k, v in self.extra.items()]
        return ";".join(kv)

    @property
    def T(self) -> int:
        return self.B * self.S

    # --- the BASELINE.json configs (SURVEY.md §8 notation) ---
    @staticmethod
    def tiny(**kw):  # C1: tiny BERT fp32 SGD (A=2, F=512, V=1024 assumed)
        return ModelConfig(**{**dict(kind="bert", L=2, H=128, A=2, F=512, V=1024, S=128, B=8,
                                     dtype="f32", opt="sgd", lr=0.01), **kw})

    @staticmethod
    def bert_base(**kw):  # C2: BERT-base MLM, bf16 AutoCast + Adam
        return ModelConfig(**{**dict(kind="bert", L=12, H=768, A=12, F=3072, V=30522, S=128, B=32,
                                     dtype="bf16", opt="adam", lr=1e-4, eps=1e-6, p=0.1), **kw})

    @staticmethod
    def bert_large(**kw):  # C4
        return ModelConfig(**{**dict(kind="bert", L=24, H=1024, A=16, F=4096, V=30522, S=128, B=32,
                                     dtype="bf16", opt="adam", lr=1e-4, eps=1e-6, p=0.1), **kw})

    @staticmethod
    def gpt2_medium(**kw):  # C3
        return ModelConfig(**{**dict(kind="gpt2", L=24, H=1024, A=16, F=4096, V=50257, S=512, B=8,
                                     dtype="bf16", opt="adam", lr=1e-4, eps=1e-6, p=0.1), **kw})

    @staticmethod
    def gpt2_xl(**kw):  # C5
        return ModelConfig(**{**dict(kind="gpt2", L=48, H=1600, A=25, F=6400, V=50257, S=1024, B=8,
                                     dtype="bf16", opt="adam", lr=1e-4, eps=1e-6, p=0.1), **kw})


def synthetic_batch(cfg: ModelConfig, seed: int | None = None):
    """SURVEY.md §8d synthetic data via trainc::Rng (MLM: 15% labelled;
    causal LM: next-token labels)."""
    T = cfg.T
    ids = np.empty(T, np.int32)
    labels = np.empty(T, np.int32)
    _check(lib().tb_synthetic_batch(T, cfg.V, cfg.seed_d if seed is None else seed, ids.ctypes.data,
                                    labels.ctypes.data, int(cfg.kind == "gpt2")))
    return ids, labels


def plan_fits(cfg: ModelConfig, budget: int, remat: bool) -> tuple[bool, dict]:
    """CPU planner: does the step at cfg fit `budget` device bytes (static
    arena + parameter/optimizer state)?  With remat, the rematerialisation pass
     runs under the budget first; an infeasible plan
    (no evictable tensor) does not fit."""
    c = ModelConfig(**{f.name: getattr(cfg, f.name) for f in fields(cfg) if f.name != "extra"})
    c.extra = dict(cfg.extra)
    c.extra.setdefault("schedule", 1)  # p-c list schedule before remat
    if remat:
        # the remat pass bounds the liveness peak; address packing of the arena
        # adds fragmentation on top, so it aims 1.5% below the budget
        c.extra["budget"] = int(budget * 0.985)
    # the greedy remat pass is not monotone in its candidate set: plan with
    # depth-2 chains through tuple producers, and without them if that fails
    tries = [1, 0] if remat and "remat_chain" not in c.extra else [c.extra.get("remat_chain", 1)]
    gi = {}
    for rc in tries:
        c.extra["remat_chain"] = rc
        try:
            gi = graph_info(c)
        except RuntimeError:
            continue
        if gi["arena_plan_bytes"] + gi["state_bytes"] <= budget:
            return True, gi
    return False, gi


def max_batch_under_remat(factory, budget: int, b0: int = 32, remat: bool = True,
                          reserve_per_sample: int = 0) -> tuple[int, dict]:
    """Largest per-GPU batch the planner fits in `budget` bytes: doubling from
    b0, then bisection ('double B until BudgetInfeasible,
    then bisect').  reserve_per_sample: bytes per sample kept outside the
    planned arena for the kernels' own batch-proportional scratch (partial
    sums, sort buffers), so the arena budget at batch B is budget - B * reserve.
    Returns (B, graph_info at B)."""
    fits = lambda B: plan_fits(factory(B=B), budget - B * reserve_per_sample, remat)  # noqa: E731
    ok, gi = fits(b0)
    if not ok:
        return 0, {}
    lo, hi, best = b0, None, gi
    while hi is None:
        ok, g = fits(lo * 2)
        if ok:
            lo, best = lo * 2, g
        else:
            hi = lo * 2
    while hi - lo > 1:
        mid = (lo + hi) // 2
        ok, g = fits(mid)
        if ok:
            lo, best = mid, g
        else:
            hi = mid
    return lo, best


INFO_FIELDS = ["P", "P_pad", "T", "arena_bytes", "state_bytes", "planner_peak", "instructions",
               "kernels_per_step", "lets", "fused_dact", "fused_ln_dy2", "fused_emb", "dead",
               "remat_replays", "peak_before_remat", "compile_us", "shard"]
GRAPH_FIELDS = ["P", "P_pad", "lets", "planner_peak", "arena_plan_bytes", "state_bytes", "fused_dact",
                "fused_ln_dy2", "fused_emb", "dead", "remat_replays", "peak_before_remat",
                "peak_after_remat", "fused_ln_bias", "fused_pairs"]


def graph_info(cfg: ModelConfig) -> dict:
    """CPU-only: build + plan the step graph without a device."""
    out = (ctypes.c_int64 * len(GRAPH_FIELDS))()
    _check(lib().tb_graph_info(cfg.cfg_string().encode(), out, len(GRAPH_FIELDS)))
    return dict(zip(GRAPH_FIELDS, list(out)))


def graph_text(cfg: ModelConfig, what: str = "ir") -> str:
    t = lib().tb_graph_text(cfg.cfg_string().encode(), what.encode()).decode()
    if not t:
        raise RuntimeError(lib().tb_last_error().decode())
    return t


def graph_segments(cfg: ModelConfig) -> list[tuple[str, int, int]]:
    """CPU-only: the flat parameter segments (name, offset, numel) of cfg's step."""
    out = []
    for line in graph_text(cfg, "segments").splitlines():
        n, o, k = line.split()
        out.append((n, int(o), int(k)))
    return out


def derive_priorities(samples: list[tuple[str, str, str, float]]) -> dict:
    """backends::derive_priorities (backends.hpp:387-419): (dialect, op,
    shape_class, median_us) samples -> {"dialect.op": priority}."""
    text = "".join(f"{d} {o} {c} {us!r}\n" for d, o, c, us in samples)
    t = lib().tb_derive_priorities(text.encode())
    if t is None:
        raise RuntimeError(lib().tb_last_error().decode())
    return {k: int(v) for k, v in (line.split() for line in t.decode().splitlines())}


def memsched_text(text: str, what: str, budget: int = 0, transient_inputs: bool = False) -> str:
    """CPU-only memsched queries on a text-IR function (tb_memsched_text)."""
    t = lib().tb_memsched_text(text.encode(), what.encode(), budget, int(transient_inputs))
    if t is None:
        raise RuntimeError(lib().tb_last_error().decode())
    return t.decode()


class Session:
    def __init__(self, cfg: ModelConfig, device: int = 0):
        self.cfg = cfg
        h = lib().tb_session_create(cfg.cfg_string().encode(), device)
        if not h:
            raise RuntimeError(lib().tb_last_error().decode())
        self.h = h
        self.T = cfg.T

    def info(self) -> dict:
        out = (ctypes.c_int64 * len(INFO_FIELDS))()
        _check(lib().tb_session_info(self.h, out, len(INFO_FIELDS)))
        return dict(zip(INFO_FIELDS, list(out)))

    def init_params(self):
        _check(lib().tb_session_init_params(self.h))

    def set_batch(self, ids: np.ndarray, labels: np.ndarray):
        ids = np.ascontiguousarray(ids, np.int32)
        labels = np.ascontiguousarray(labels, np.int32)
        _check(lib().tb_session_set_batch(self.h, ids.ctypes.data, labels.ctypes.data))

    def staging(self):
        """numpy views of the pinned host staging buffers (ids, labels)."""
        L = lib()
        T = self.T
        ids = np.ctypeslib.as_array((ctypes.c_int32 * T).from_address(L.tb_session_ids_buffer(self.h)))
        lab = np.ctypeslib.as_array((ctypes.c_int32 * T).from_address(L.tb_session_labels_buffer(self.h)))
        return ids, lab

    def set_batch_from_staging(self):
        L = lib()
        _check(L.tb_session_set_batch(self.h, L.tb_session_ids_buffer(self.h), L.tb_session_labels_buffer(self.h)))

    def step(self, graph: bool = True):
        _check(lib().tb_session_step(self.h, int(graph)))

    def fetch_loss(self):
        _check(lib().tb_session_fetch_loss(self.h))

    def sync(self):
        _check(lib().tb_session_sync(self.h))

    def loss(self) -> float:
        self.fetch_loss()
        self.sync()
        return float(lib().tb_session_loss_value(self.h))

    @property
    def stream(self) -> int:
        return lib().tb_session_stream(self.h)

    def param_ptr(self, name: str):
        p = ctypes.c_void_p()
        n = ctypes.c_int64()
        _check(lib().tb_session_param(self.h, name.encode(), ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def read(self, name: str, dtype=np.float32) -> np.ndarray:
        ptr, nbytes = self.param_ptr(name)
        out = np.empty(nbytes // np.dtype(dtype).itemsize, dtype)
        self.sync()
        runtime.check(runtime.lib().tcb_memcpy(ctypes.c_void_p(out.ctypes.data), ctypes.c_void_p(ptr),
                                               ctypes.c_uint64(nbytes), 1, None))
        runtime.check(runtime.lib().tcb_device_sync())
        return out

    def write(self, name: str, arr: np.ndarray):
        ptr, nbytes = self.param_ptr(name)
        arr = np.ascontiguousarray(arr)
        assert arr.nbytes == nbytes, (arr.nbytes, nbytes)
        runtime.check(runtime.lib().tcb_memcpy(ctypes.c_void_p(ptr), ctypes.c_void_p(arr.ctypes.data),
                                               ctypes.c_uint64(nbytes), 0, None))
        runtime.check(runtime.lib().tcb_device_sync())

    def segments(self) -> list[tuple[str, int, int]]:
        out = []
        for line in lib().tb_session_segments(self.h).decode().splitlines():
            n, o, k = line.split()
            out.append((n, int(o), int(k)))
        return out

    def text(self, what: str) -> str:
        return lib().tb_session_text(self.h, what.encode()).decode()

    def profile(self, repeats: int = 5, inner: int = 1) -> list[dict]:
        """vm.profile: per-instruction median device time of
        eager steps (CUDA events around every instruction and fold flush).
        inner > 1 runs each launch that many times back to back between its
        events and reports the mean (no per-launch event round trip); it
        advances the training state `inner` updates per profiled step."""
        t = lib().tb_session_profile_inner(self.h, repeats, inner)
        if t is None:
            raise RuntimeError(lib().tb_last_error().decode())
        rows = []
        lines = t.decode().splitlines()
        for line in lines[1:]:
            i, op, let, us, bi, bo, k, shapes = line.split(",")
            ins, _, outs = shapes.partition(">")
            parse = lambda t: [tuple(int(d) for d in x.split("x")) for x in t.split(";") if x]  # noqa: E731
            rows.append({"idx": int(i), "op": op, "let": int(let), "us": float(us), "bytes_in": int(bi),
                         "bytes_out": int(bo), "kernels": int(k), "in": parse(ins), "out": parse(outs)})
        return rows

    def set_comm(self, comm: int):
        _check(lib().tb_session_set_comm(self.h, comm))

    STATE = ("params", "p16", "m", "v", "step", "rng_step")

    def state_names(self) -> list[str]:
        """Training-state parameters of this step graph (master weights, the
        bf16 compute copy, Adam moments, step counter) -- what a checkpoint holds."""
        out = []
        for n in self.STATE:
            try:
                self.param_ptr(n)
            except RuntimeError:
                continue
            out.append(n)
        return out

    def save_param(self, name: str, path: str):
        """One step parameter -> TNSR file (tensor.hpp:80-104 layout; bf16 code 2)."""
        _check(lib().tb_session_save_param(self.h, name.encode(), os.fsencode(path)))

    def load_param(self, name: str, path: str):
        """TNSR file -> step parameter (dtype code and shape must match)."""
        _check(lib().tb_session_load_param(self.h, name.encode(), os.fsencode(path)))

    def save_checkpoint(self, directory: str) -> list[str]:
        """Write the training state as <directory>/<name>.tnsr, one file per state
        parameter; on ZeRO ranks each rank writes its own shard (name.rank<r>)."""
        os.makedirs(directory, exist_ok=True)
        names = self.state_names()
        sfx = f".rank{self.cfg.extra.get('rank', 0)}" if self.cfg.world > 1 else ""
        for n in names:
            self.save_param(n, os.path.join(directory, f"{n}{sfx}.tnsr"))
        return names

    def load_checkpoint(self, directory: str) -> list[str]:
        names = self.state_names()
        sfx = f".rank{self.cfg.extra.get('rank', 0)}" if self.cfg.world > 1 else ""
        for n in names:
            self.load_param(n, os.path.join(directory, f"{n}{sfx}.tnsr"))
        return names

    def close(self):
        if getattr(self, "h", None):
            lib().tb_session_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


TNSR_CODES = {np.dtype(np.float32): 0, np.dtype(np.float16): 1, np.dtype(np.int32): 3}
TNSR_DTYPES = {0: np.float32, 1: np.float16, 2: np.uint16, 3: np.int32}  # 2 = bf16 bits


def tnsr_save(path: str, arr: np.ndarray, code: int | None = None):
    """Host array -> TNSR file through the native writer (host/tnsr.hpp).
    bf16 is passed as uint16 bit patterns with code=2."""
    arr = np.require(arr, requirements="C")  # keeps rank 0 (ascontiguousarray would not)
    if code is None:
        code = TNSR_CODES[arr.dtype]
    if np.dtype(TNSR_DTYPES[code]).itemsize != arr.itemsize:
        raise TypeError(f"array dtype {arr.dtype} does not match TNSR code {code}")
    shape = (ctypes.c_int64 * max(arr.ndim, 1))(*arr.shape)
    _check(lib().tb_tnsr_save(os.fsencode(path), arr.ctypes.data, code, arr.ndim, shape))


def tnsr_load(path: str) -> tuple[np.ndarray, int]:
    """TNSR file -> (array, code) through the native reader."""
    code, rank = ctypes.c_int(), ctypes.c_int()
    shape = (ctypes.c_int64 * 255)()
    _check(lib().tb_tnsr_header(os.fsencode(path), ctypes.byref(code), ctypes.byref(rank), shape, 255))
    out = np.empty(tuple(shape[:rank.value]), TNSR_DTYPES[code.value])
    _check(lib().tb_tnsr_load(os.fsencode(path), out.ctypes.data, out.nbytes))
    return out, code.value


def cache_stats() -> dict:
    out = (ctypes.c_int64 * 3)()
    _check(lib().tb_cache_stats(out))
    return {"compiles": out[0], "hits": out[1], "size": out[2]}


def cache_clear():
    """Drop every compiled plan and its device scratch (KernelCache::clear,
    backends.hpp:356-361).  Call only with no Session alive."""
    _check(lib().tb_cache_clear())


AUTOCAST_FIELDS = ("sites", "casts", "exclusive", "shared", "low_ops", "f32_violations", "standalone_casts",
                   "param_casts", "lets")


def autocast_info(cfg: "ModelConfig", policy: str = "b200", placement: str = "auto") -> dict:
    """Run the AutoCast pass on the all-f32 training step of `cfg` (CPU only)
    and return its cast census (host/autocast.hpp)."""
    out = (ctypes.c_int64 * len(AUTOCAST_FIELDS))()
    _check(lib().tb_autocast_info(cfg.cfg_string(model_only=True).encode(), policy.encode(), placement.encode(),
                                  out, len(AUTOCAST_FIELDS)))
    return dict(zip(AUTOCAST_FIELDS, list(out)))


def text_reprint(text: str) -> str:
    """Parse text IR (the reference format + bf16/i32 tokens) and print it again."""
    t = lib().tb_text_reprint(text.encode())
    if t is None:
        raise RuntimeError(lib().tb_last_error().decode())
    return t.decode()


def train_report(cfg: "ModelConfig", steps: int, path: str | None = None, seed: int | None = None,
                 graph: bool = True) -> list[tuple[int, float, float, int]]:
    """`trainc train --report out.csv`: run `steps` training
    steps on synthetic data from `seed` and return / write rows of
    (step, loss, iter_time, peak_pool_bytes).  iter_time is the step's device
    time in seconds (CUDA events on the session stream); peak_pool_bytes is the
    static arena + state the memory planner reserved (the VM never allocates
    inside a step).  Same seed -> identical loss column."""
    from . import runtime as R
    s = Session(cfg)
    rows = []
    try:
        s.init_params()
        info = s.info()
        pool = int(info["arena_bytes"]) + int(info["state_bytes"])
        L = R.lib()
        ev0, ev1 = ctypes.c_void_p(), ctypes.c_void_p()
        R.check(L.tcb_event_create(ctypes.byref(ev0)))
        R.check(L.tcb_event_create(ctypes.byref(ev1)))
        for k in range(steps):
            ids, labels = synthetic_batch(cfg, seed=(cfg.seed_d if seed is None else seed) + k)
            s.set_batch(ids, labels)
            R.check(L.tcb_event_record(ev0, ctypes.c_void_p(s.stream)))
            s.step(graph=graph)
            R.check(L.tcb_event_record(ev1, ctypes.c_void_p(s.stream)))
            loss = s.loss()
            ms = ctypes.c_float()
            R.check(L.tcb_event_elapsed_ms(ev0, ev1, ctypes.byref(ms)))
            rows.append((k, loss, ms.value * 1e-3, pool))
        L.tcb_event_destroy(ev0)
        L.tcb_event_destroy(ev1)
    finally:
        s.close()
    if path is not None:
        with open(path, "w") as f:
            f.write("step,loss,iter_time,peak_pool_bytes\n")
            for k, loss, t, pool in rows:
                f.write(f"{k},{float(loss):.9g},{t:.6e},{pool}\n")  # 9 digits round-trip an f32
    return rows
