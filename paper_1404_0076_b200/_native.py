"""ctypes binding of libinetb200.so (include/inet_b200.h).

The library is built in-tree (``python __graft_entry__.py`` or
``make -C paper_1404_0076_b200/csrc``). There is no fallback: if the shared
object is missing or no CUDA device is visible, the engine raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import DeviceError

LIB_PATH = os.environ.get("INET_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)),
                                                             "libinetb200.so")

OK, NO_RULE, LOOP_CAP, ARENA, CUDA, ARG, UNSUPPORTED, NO_DEVICE, STATE, NAME, ORDER = range(11)

EXPORTS = (
    "inet_ctx_create",
    "inet_ctx_destroy",
    "inet_strerror",
    "inet_abi_sizes",
    "inet_device_info",
    "inet_rules_load",
    "inet_set_jit",
    "inet_jit_compile",
    "inet_jit_precompile",
    "inet_batch_load",
    "inet_batch_reduce",
    "inet_batch_rerun",
    "inet_batch_collect",
    "inet_batch_stats_all",
    "inet_batch_result_counts",
    "inet_batch_print_all",
    "inet_batch_stats",
    "inet_batch_rule_counts",
    "inet_batch_io_bytes",
    "inet_batch_totals",
    "inet_batch_rounds",
    "inet_batch_finalize",
    "inet_batch_result",
    "inet_finalize_flat",
    "inet_print_flat",
    "inet_batch_print",
)


class Cfg(C.Structure):
    _fields_ = [
        ("max_loops", C.c_uint32),
        ("collect_stats", C.c_uint32),
        ("threads", C.c_uint32),
        ("ctas_per_net", C.c_uint32),
        ("cap_agents", C.c_uint32),
        ("cap_vars", C.c_uint32),
        ("max_retries", C.c_uint32),
        ("count_rules", C.c_uint32),
        ("exact_loops", C.c_uint32),
        ("reference_order", C.c_uint32),
        ("validate_phases", C.c_uint32),
        ("var_order", C.c_uint32),
    ]


class NetStats(C.Structure):
    _fields_ = [
        ("interactions", C.c_uint64),
        ("communications", C.c_uint64),
        ("rounds", C.c_uint32),
        ("status", C.c_uint32),
        ("err_label_a", C.c_uint32),
        ("err_label_b", C.c_uint32),
        ("agent_hw", C.c_uint32),
        ("var_hw", C.c_uint32),
        ("n_residual", C.c_uint32),
        ("cap_agents", C.c_uint32),
        ("cap_vars", C.c_uint32),
        ("tier", C.c_uint32),
        ("jit", C.c_uint32),
        ("sm_mhz", C.c_uint32),
        ("device_final", C.c_uint32),
        ("threads", C.c_uint32),
    ]


_lib = None
_lib_lock = threading.Lock()

_u32p = C.POINTER(C.c_uint32)
_u64p = C.POINTER(C.c_uint64)


def _choose_nvrtc() -> None:
    """Point the rule-set compiler at the NVRTC that ships with torch's CUDA
    runtime (the `nvidia-cuda-nvrtc` wheel) when it is installed, so the
    compiler does not depend on which libnvrtc.so.12 a process loaded first.
    Its code measured faster than the system toolkit's on the shipped
    programs. INET_B200_NVRTC set by the user wins."""
    if os.environ.get("INET_B200_NVRTC"):
        return
    try:
        import nvidia.cuda_nvrtc as nv
    except ImportError:
        return
    for base in getattr(nv, "__path__", []):
        cand = os.path.join(base, "lib", "libnvrtc.so.12")
        if os.path.exists(cand):
            os.environ["INET_B200_NVRTC"] = cand
            return


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """Load the shared object and declare every exported signature."""
    global _lib
    with _lib_lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(-1, f"native library not built: {path} (run `python __graft_entry__.py`)")
        _choose_nvrtc()
        lib = C.CDLL(path)
        sig = {
            "inet_ctx_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
            "inet_ctx_destroy": (None, [C.c_void_p]),
            "inet_strerror": (C.c_char_p, [C.c_int]),
            "inet_abi_sizes": (None, [C.POINTER(C.c_size_t), C.POINTER(C.c_size_t)]),
            "inet_device_info": (C.c_int, [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.c_char_p, C.c_size_t]),
            "inet_rules_load": (C.c_int, [C.c_void_p, _u32p, C.c_size_t]),
            "inet_set_jit": (C.c_int, [C.c_void_p, C.c_int]),
            "inet_jit_compile": (C.c_int, [_u32p, C.c_size_t, C.c_int, C.c_uint32, C.c_char_p, C.c_size_t]),
            "inet_jit_precompile": (
                C.c_int, [_u32p, C.c_size_t, C.c_int, C.c_uint32, C.c_uint32, C.c_char_p, C.c_size_t]),
            "inet_batch_load": (C.c_int, [C.c_void_p, C.c_uint32, _u32p, _u64p, _u32p, _u64p, _u32p, _u64p, _u32p]),
            "inet_batch_reduce": (C.c_int, [C.c_void_p, C.POINTER(Cfg), C.POINTER(C.c_float)]),
            "inet_batch_rerun": (C.c_int, [C.c_void_p, C.POINTER(Cfg), C.POINTER(C.c_float)]),
            "inet_batch_collect": (C.c_int, [C.c_void_p]),
            "inet_batch_stats_all": (C.c_int, [C.c_void_p, C.POINTER(NetStats), C.c_uint32]),
            "inet_batch_result_counts": (C.c_int, [C.c_void_p, _u32p, _u32p, _u32p, C.c_uint32]),
            "inet_batch_print_all": (C.c_int, [C.c_void_p, C.POINTER(C.c_char_p), C.POINTER(C.c_uint8), C.c_uint32,
                                               C.c_uint32, C.c_char_p, C.c_size_t, _u64p,
                                               C.POINTER(C.c_size_t)]),
            "inet_batch_stats": (C.c_int, [C.c_void_p, C.c_uint32, C.POINTER(NetStats)]),
            "inet_batch_totals": (C.c_int, [C.c_void_p, _u64p, _u64p, _u32p, _u32p]),
            "inet_batch_rule_counts": (C.c_int, [C.c_void_p, C.c_uint32, _u64p, C.c_uint32]),
            "inet_batch_io_bytes": (C.c_int, [C.c_void_p, _u64p, _u64p]),
            "inet_batch_rounds": (C.c_int, [C.c_void_p, C.c_uint32, _u32p, _u32p]),
            "inet_batch_finalize": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32]),
            "inet_batch_result": (
                C.c_int,
                [C.c_void_p, C.c_uint32, C.POINTER(_u32p), _u32p, C.POINTER(_u32p), _u32p, C.POINTER(_u32p), _u32p],
            ),
            "inet_finalize_flat": (
                C.c_int,
                [_u32p, C.c_uint32, _u32p, C.c_uint32, _u32p, C.c_uint32, C.c_uint32, C.POINTER(C.c_uint8)],
            ),
            "inet_print_flat": (
                C.c_int,
                [_u32p, C.c_uint32, _u32p, C.c_uint32, _u32p, C.c_uint32, C.POINTER(C.c_char_p),
                 C.POINTER(C.c_uint8), C.c_uint32, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
            ),
            "inet_batch_print": (
                C.c_int,
                [C.c_void_p, C.c_uint32, C.POINTER(C.c_char_p), C.POINTER(C.c_uint8), C.c_uint32, C.c_char_p,
                 C.c_size_t, C.POINTER(C.c_size_t)],
            ),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        cfg_b, st_b = C.c_size_t(), C.c_size_t()
        lib.inet_abi_sizes(C.byref(cfg_b), C.byref(st_b))
        if cfg_b.value != C.sizeof(Cfg) or st_b.value != C.sizeof(NetStats):
            raise DeviceError(-1, f"ABI mismatch: inet_cfg {cfg_b.value} vs {C.sizeof(Cfg)} bytes, "
                                  f"inet_net_stats {st_b.value} vs {C.sizeof(NetStats)} bytes")
        _lib = lib
        return lib


def strerror(code: int) -> str:
    return load_library().inet_strerror(code).decode()


def _ptr(a: np.ndarray, ctype=C.c_uint32):
    return a.ctypes.data_as(C.POINTER(ctype))


def _check(code: int, what: str) -> None:
    if code not in (OK, NO_RULE, LOOP_CAP, ARENA, NAME, ORDER):
        raise DeviceError(code, f"{what}: {strerror(code)}")


class Context:
    """One device, one stream; device buffers persist across calls."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = C.c_void_p()
        code = lib.inet_ctx_create(device, C.byref(h))
        if code != OK:
            raise DeviceError(code, f"inet_ctx_create(device={device}): {strerror(code)}")
        self.lib = lib
        self.h = h
        self.device = device
        self.lock = threading.Lock()
        self._blob_key = None

    def close(self):
        if self.h:
            self.lib.inet_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        sms, clk = C.c_int(), C.c_int()
        name = C.create_string_buffer(128)
        _check(self.lib.inet_device_info(self.h, C.byref(sms), C.byref(clk), name, 128), "device_info")
        return {"sm_count": sms.value, "clock_khz": clk.value, "name": name.value.decode()}

    def set_jit(self, mode: bool) -> None:
        """Rule-set specialised kernels on/off (default on when NVRTC is present)."""
        _check(self.lib.inet_set_jit(self.h, 1 if mode else 0), "set_jit")

    def load_rules(self, blob: np.ndarray, key=None) -> None:
        if key is not None and key == self._blob_key:
            return
        blob = np.ascontiguousarray(blob, dtype=np.uint32)
        _check(self.lib.inet_rules_load(self.h, _ptr(blob), blob.size), "rules_load")
        self._blob_key = key

    def load_batch(self, agents, agent_off, eqs, eq_off, iface, iface_off, n_vars) -> None:
        agents = np.ascontiguousarray(agents, dtype=np.uint32).reshape(-1)
        eqs = np.ascontiguousarray(eqs, dtype=np.uint32).reshape(-1)
        iface = np.ascontiguousarray(iface, dtype=np.uint32).reshape(-1)
        agent_off = np.ascontiguousarray(agent_off, dtype=np.uint64)
        eq_off = np.ascontiguousarray(eq_off, dtype=np.uint64)
        iface_off = np.ascontiguousarray(iface_off, dtype=np.uint64)
        n_vars = np.ascontiguousarray(n_vars, dtype=np.uint32)
        n = len(n_vars)
        # keep a non-empty buffer so pointers are valid
        agents = agents if agents.size else np.zeros(4, np.uint32)
        eqs = eqs if eqs.size else np.zeros(2, np.uint32)
        iface = iface if iface.size else np.zeros(1, np.uint32)
        code = self.lib.inet_batch_load(
            self.h, n, _ptr(agents), _ptr(agent_off, C.c_uint64), _ptr(eqs), _ptr(eq_off, C.c_uint64),
            _ptr(iface), _ptr(iface_off, C.c_uint64), _ptr(n_vars),
        )
        _check(code, "batch_load")

    def reduce(self, cfg: Cfg) -> tuple[int, float]:
        ms = C.c_float()
        code = self.lib.inet_batch_reduce(self.h, C.byref(cfg), C.byref(ms))
        _check(code, "batch_reduce")
        return code, ms.value

    def rerun(self, cfg: Cfg) -> float:
        ms = C.c_float()
        _check(self.lib.inet_batch_rerun(self.h, C.byref(cfg), C.byref(ms)), "batch_rerun")
        return ms.value

    def collect(self) -> int:
        """Statistics and results of the last launch (e.g. the last timed rerun)."""
        code = self.lib.inet_batch_collect(self.h)
        _check(code, "batch_collect")
        return code

    def stats_all(self, n: int) -> list:
        """Every net's NetStats in one call."""
        arr = (NetStats * max(n, 1))()
        _check(self.lib.inet_batch_stats_all(self.h, arr, n), "batch_stats_all")
        return list(arr)[:n]

    def result_counts_all(self, n: int) -> np.ndarray:
        """(n, 3) agents / interface terms / equations of every finalized net's normal form."""
        out = np.zeros((3, max(n, 1)), dtype=np.uint32)
        _check(self.lib.inet_batch_result_counts(self.h, _ptr(out[0]), _ptr(out[1]), _ptr(out[2]), n),
               "batch_result_counts")
        return out[:, :n].T

    def texts(self, n: int, labels: "LabelTable", threads: int = 0) -> list:
        """Canonical text of every finalized net (printed natively, in parallel)."""
        names, arity, nl = labels.args()
        size = C.c_size_t()
        _check(self.lib.inet_batch_print_all(self.h, names, arity, nl, threads, None, 0, None, C.byref(size)),
               "batch_print_all")
        buf = C.create_string_buffer(max(size.value, 1))
        offs = np.zeros(n + 1, dtype=np.uint64)
        _check(self.lib.inet_batch_print_all(self.h, names, arity, nl, threads, buf, size.value,
                                             _ptr(offs, C.c_uint64), C.byref(size)), "batch_print_all")
        raw = buf.raw[: size.value].decode()
        o = offs.tolist()
        return [raw[o[i]:o[i + 1]] for i in range(n)]

    def stats(self, net: int) -> NetStats:
        s = NetStats()
        _check(self.lib.inet_batch_stats(self.h, net, C.byref(s)), "batch_stats")
        return s

    def rule_counts(self, net: int, n_rules: int) -> np.ndarray:
        out = np.zeros(max(n_rules, 1), dtype=np.uint64)
        _check(self.lib.inet_batch_rule_counts(self.h, net, _ptr(out, C.c_uint64), n_rules), "rule_counts")
        return out[:n_rules]

    def io_bytes(self) -> tuple[int, int]:
        h2d, d2h = C.c_uint64(), C.c_uint64()
        _check(self.lib.inet_batch_io_bytes(self.h, C.byref(h2d), C.byref(d2h)), "io_bytes")
        return h2d.value, d2h.value

    def totals(self) -> tuple[int, int, int, int]:
        ti, tc, mr, nf = C.c_uint64(), C.c_uint64(), C.c_uint32(), C.c_uint32()
        _check(self.lib.inet_batch_totals(self.h, C.byref(ti), C.byref(tc), C.byref(mr), C.byref(nf)), "totals")
        return ti.value, tc.value, mr.value, nf.value

    def rounds(self, net: int) -> np.ndarray:
        n = C.c_uint32()
        _check(self.lib.inet_batch_rounds(self.h, net, None, C.byref(n)), "batch_rounds")
        rows = np.zeros((max(n.value, 1), 4), dtype=np.uint32)
        _check(self.lib.inet_batch_rounds(self.h, net, _ptr(rows), C.byref(n)), "batch_rounds")
        return rows[: n.value]

    def finalize(self, net: int = 0xFFFFFFFF, threads: int = 0) -> int:
        code = self.lib.inet_batch_finalize(self.h, net, threads)
        if code not in (OK,):
            raise DeviceError(code, f"batch_finalize: {strerror(code)}")
        return code

    def text(self, net: int, labels: "LabelTable") -> str:
        """Canonical text of a finalized net, printed natively."""
        names, arity, nl = labels.args()
        return _print_call(lambda b, cap, n: self.lib.inet_batch_print(self.h, net, names, arity, nl, b, cap, n),
                           "batch_print")

    def result_counts(self, net: int) -> tuple[int, int, int]:
        """(agents, interface terms, equations) of a finalized net's normal form, no copies."""
        na, ni, ne = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(self.lib.inet_batch_result(self.h, net, None, C.byref(na), None, C.byref(ni), None, C.byref(ne)),
               "batch_result")
        return na.value, ni.value, ne.value

    def result(self, net: int) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        pa, pi, pe = _u32p(), _u32p(), _u32p()
        na, ni, ne = C.c_uint32(), C.c_uint32(), C.c_uint32()
        code = self.lib.inet_batch_result(
            self.h, net, C.byref(pa), C.byref(na), C.byref(pi), C.byref(ni), C.byref(pe), C.byref(ne)
        )
        _check(code, "batch_result")

        def grab(p, n, width):
            if n == 0:
                return np.zeros((0, width), dtype=np.uint32) if width > 1 else np.zeros(0, dtype=np.uint32)
            arr = np.ctypeslib.as_array(p, shape=(n * width,)).copy()
            return arr.reshape(n, width) if width > 1 else arr

        return grab(pa, na.value, 4), grab(pi, ni.value, 1), grab(pe, ne.value, 2)


def finalize_flat(agents: np.ndarray, iface: np.ndarray, eqs: np.ndarray, n_vars: int):
    """In-place host finalize on flat arrays; returns the alive mask."""
    lib = load_library()
    agents = np.ascontiguousarray(agents, dtype=np.uint32)
    iface = np.ascontiguousarray(iface, dtype=np.uint32)
    eqs = np.ascontiguousarray(eqs, dtype=np.uint32)
    alive = np.zeros(max(len(eqs.reshape(-1)) // 2, 1), dtype=np.uint8)
    code = lib.inet_finalize_flat(
        _ptr(agents), len(agents.reshape(-1)) // 4, _ptr(iface), iface.size, _ptr(eqs), len(eqs.reshape(-1)) // 2,
        n_vars, alive.ctypes.data_as(C.POINTER(C.c_uint8)),
    )
    if code != OK:
        raise DeviceError(code, f"finalize_flat: {strerror(code)}")
    return agents, iface, eqs, alive[: len(eqs.reshape(-1)) // 2]


class LabelTable:
    """Label names and arities in the C layout the printer takes."""

    def __init__(self, names, arities):
        self._raw = [n.encode() for n in names]
        self.names = (C.c_char_p * max(len(names), 1))(*self._raw)
        self.arity = np.ascontiguousarray(arities, dtype=np.uint8)
        self.n = len(names)

    def args(self):
        return self.names, self.arity.ctypes.data_as(C.POINTER(C.c_uint8)), self.n


def _print_call(call, what: str) -> str:
    n = C.c_size_t()
    buf = C.create_string_buffer(1 << 16)
    code = call(buf, len(buf), C.byref(n))
    _check(code, what)
    if n.value > len(buf):
        buf = C.create_string_buffer(n.value)
        code = call(buf, len(buf), C.byref(n))
        _check(code, what)
    return buf.raw[: n.value].decode()


def print_flat(agents: np.ndarray, iface: np.ndarray, eqs: np.ndarray, labels: LabelTable) -> str:
    """Canonical text (lang.print_configuration) of a flat normal form."""
    lib = load_library()
    agents = np.ascontiguousarray(agents, dtype=np.uint32).reshape(-1)
    iface = np.ascontiguousarray(iface, dtype=np.uint32).reshape(-1)
    eqs = np.ascontiguousarray(eqs, dtype=np.uint32).reshape(-1)
    names, arity, nl = labels.args()
    return _print_call(
        lambda b, cap, n: lib.inet_print_flat(_ptr(agents), agents.size // 4, _ptr(iface), iface.size, _ptr(eqs),
                                              eqs.size // 2, names, arity, nl, b, cap, n),
        "print_flat")


def jit_compile(blob: np.ndarray, tier: int = 1, threads: int = 1024) -> tuple[int, str]:
    """Compile the rule-set specialised kernel on the host (no device needed)."""
    lib = load_library()
    blob = np.ascontiguousarray(blob, dtype=np.uint32)
    log = C.create_string_buffer(1 << 16)
    code = lib.inet_jit_compile(_ptr(blob), blob.size, tier, threads, log, len(log))
    return code, log.value.decode(errors="replace")


TIER_S, TIER_M, TIER_G, TIER_C, TIER_X, TIER_R = 0, 1, 2, 3, 4, 5


def jit_precompile(blob: np.ndarray, tier: int, threads: int, exact_code: bool, count_rules: bool,
                   stamps: bool = False, style: int = -1, rows: bool = True) -> tuple[int, str]:
    """Compile one kernel variant into the package's kernels/ directory (build time)."""
    lib = load_library()
    blob = np.ascontiguousarray(blob, dtype=np.uint32)
    log = C.create_string_buffer(1 << 16)
    flags = (1 if exact_code else 0) | (2 if count_rules else 0) | (4 if stamps else 0) | (0 if rows else 8) | ((style + 1) << 8)
    code = lib.inet_jit_precompile(_ptr(blob), blob.size, tier, threads, flags, log, len(log))
    return code, log.value.decode(errors="replace")


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    """Process-wide context per device (created on first use)."""
    with _lib_lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lib_lock:
            _contexts.setdefault(device, ctx)
            ctx = _contexts[device]
    return ctx
