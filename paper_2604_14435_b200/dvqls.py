"""Thin ctypes binding of libdvqls.so (include/dvqls.h), same names as the C ABI.

Argument marshalling only: every step of the hot path runs in the library's
sm_100a kernels.  There is no CPU fallback; if the in-tree ``libdvqls.so`` is
missing or the device is not an sm_100 part the calls raise.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdvqls.so")

DVQLS_OK = 0
DVQLS_E_ARG = -1
DVQLS_E_PAULI = -2
DVQLS_E_BPREP = -3
DVQLS_E_DEGENERATE = -4
DVQLS_E_CUDA = -5
DVQLS_E_NCCL = -6
DVQLS_E_UNSUPPORTED = -7
DVQLS_B_UNIFORM = 0
DVQLS_B_AMPLITUDES = 1
DVQLS_MODE_CIRCUITS = 0
DVQLS_MODE_PAULI = 1
DVQLS_ALLREDUCE_P2P = 0
DVQLS_ALLREDUCE_NCCL = 1

EXPORTED = [
    "dvqls_create", "dvqls_destroy", "dvqls_terms", "dvqls_cost", "dvqls_cost_batch",
    "dvqls_cost_dev", "dvqls_terms_local_dev", "dvqls_last_error", "dvqls_num_circuits",
    "dvqls_local_range", "dvqls_stream", "dvqls_launches_per_call", "dvqls_last_timings",
    "dvqls_nccl_unique_id", "dvqls_build_info", "dvqls_shard_range", "dvqls_state",
    "dvqls_terms_subset", "dvqls_launch_grid", "dvqls_num_observables", "dvqls_task_observable",
    "dvqls_costs_dev", "dvqls_global_cost", "dvqls_decompose", "dvqls_pauli_coefficients",
    "dvqls_decompose_error", "dvqls_workspace_size", "dvqls_cost_grad", "dvqls_cost_grad_dev",
    "dvqls_check", "dvqls_num_graphs",
]

# int (*host_allgather)(void* user, const void* send, void* recv, size_t bytes)
HOST_ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t)


class DvqlsError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"dvqls error {code}: {msg}")
        self.code = code


class DegenerateError(DvqlsError):
    pass


class _BPrep(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("amps", ctypes.POINTER(ctypes.c_double))]


class _Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("rank", ctypes.c_int), ("world", ctypes.c_int),
                ("nccl_unique_id", ctypes.c_void_p), ("entangler", ctypes.c_int),
                ("cuda_stream", ctypes.c_void_p), ("timing", ctypes.c_int), ("max_batch", ctypes.c_int),
                ("mode", ctypes.c_int), ("workspace_dev", ctypes.c_void_p), ("workspace_bytes", ctypes.c_size_t),
                ("virtual_rank", ctypes.c_int), ("virtual_world", ctypes.c_int), ("allreduce", ctypes.c_int),
                ("p2p_timeout_ms", ctypes.c_int), ("host_allgather", HOST_ALLGATHER),
                ("host_allgather_user", ctypes.c_void_p), ("graphs", ctypes.c_int), ("pdl", ctypes.c_int),
                ("stage", ctypes.c_int), ("stream_grid", ctypes.c_int), ("variant", ctypes.c_int),
                ("prefix", ctypes.c_int)]


def _opts(device=-1, rank=0, world=1, nccl_id=None, entangler=0, stream=None, timing=False, max_batch=16, mode=0,
          workspace=(None, 0), virtual_rank=0, virtual_world=0, allreduce=DVQLS_ALLREDUCE_P2P, p2p_timeout_ms=0,
          host_allgather=None, graphs=True, pdl=True, stage=0, stream_grid=0, variant=0, prefix=0):
    op = _Opts()
    op.device, op.rank, op.world = int(device), int(rank), int(world)
    op.nccl_unique_id = nccl_id
    op.entangler, op.cuda_stream, op.timing = int(entangler), stream, 1 if timing else 0
    op.max_batch, op.mode = int(max_batch), int(mode)
    op.workspace_dev, op.workspace_bytes = workspace[0], int(workspace[1])
    op.virtual_rank, op.virtual_world = int(virtual_rank), int(virtual_world)
    op.allreduce, op.p2p_timeout_ms = int(allreduce), int(p2p_timeout_ms)
    if host_allgather is not None:
        op.host_allgather = host_allgather
    op.graphs = 0 if graphs else -1
    op.pdl = 0 if pdl else -1
    op.stage, op.stream_grid, op.variant, op.prefix = int(stage), int(stream_grid), int(variant), int(prefix)
    return op


def make_host_allgather(group=None):
    """A host_allgather callback over torch.distributed (any backend, e.g. gloo): each rank's
    `bytes` bytes are gathered in rank order into recv (dvqls_opts.host_allgather)."""
    import torch.distributed as dist

    def _cb(user, send, recv, nbytes):
        try:
            mine = ctypes.string_at(send, nbytes)
            world = dist.get_world_size(group)
            out = [None] * world
            dist.all_gather_object(out, mine, group=group)
            for r, blob in enumerate(out):
                ctypes.memmove(recv + r * nbytes, blob, nbytes)
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed exchange
            return 1

    return HOST_ALLGATHER(_cb)


_lib = None


def load():
    """Load the in-tree libdvqls.so (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"CUDA extension missing: {LIB_PATH} (run python -m paper_2604_14435_b200.build)")
    L = ctypes.CDLL(LIB_PATH)
    dp = ctypes.POINTER(ctypes.c_double)
    vp = ctypes.c_void_p
    L.dvqls_create.argtypes = [ctypes.POINTER(vp), ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_char_p,
                               dp, ctypes.POINTER(_BPrep), ctypes.POINTER(_Opts)]
    L.dvqls_destroy.argtypes = [vp]
    L.dvqls_destroy.restype = None
    L.dvqls_terms.argtypes = [vp, dp, dp]
    # the per-call host-buffer entry points take plain addresses (c_void_p from int): building a
    # ctypes double pointer costs ~3 us per argument, a noticeable share of a K = 1 call
    L.dvqls_cost.argtypes = [vp, vp, vp, vp]
    L.dvqls_cost_batch.argtypes = [vp, ctypes.c_int, vp, vp, vp]
    L.dvqls_cost_dev.argtypes = [vp, ctypes.c_int, vp, vp]
    L.dvqls_terms_local_dev.argtypes = [vp, vp, vp]
    L.dvqls_state.argtypes = [vp, dp, dp]
    L.dvqls_terms_subset.argtypes = [vp, dp, ctypes.POINTER(ctypes.c_int64), ctypes.c_int64, dp]
    L.dvqls_last_error.argtypes = [vp]
    L.dvqls_last_error.restype = ctypes.c_char_p
    L.dvqls_num_circuits.argtypes = [vp]
    L.dvqls_num_circuits.restype = ctypes.c_int64
    L.dvqls_local_range.argtypes = [vp, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
    L.dvqls_stream.argtypes = [vp]
    L.dvqls_stream.restype = vp
    L.dvqls_launches_per_call.argtypes = [vp]
    L.dvqls_launch_grid.argtypes = [vp]
    L.dvqls_costs_dev.argtypes = [vp, ctypes.c_int, vp, vp, vp]
    L.dvqls_decompose.argtypes = [ctypes.c_int, dp, ctypes.c_double, ctypes.c_int64, ctypes.c_char_p, dp,
                                  ctypes.POINTER(ctypes.c_int64), dp, ctypes.c_int, ctypes.POINTER(ctypes.c_float)]
    L.dvqls_pauli_coefficients.argtypes = [ctypes.c_int, dp, dp, ctypes.c_int]
    L.dvqls_decompose_error.restype = ctypes.c_char_p
    L.dvqls_global_cost.argtypes = [vp, dp, dp, dp]
    L.dvqls_num_observables.argtypes = [vp]
    L.dvqls_num_observables.restype = ctypes.c_int64
    u32p = ctypes.POINTER(ctypes.c_uint32)
    L.dvqls_task_observable.argtypes = [ctypes.c_int, ctypes.c_char_p, ctypes.c_char_p, ctypes.c_int, u32p, u32p,
                                        ctypes.POINTER(ctypes.c_int)]
    L.dvqls_last_timings.argtypes = [vp, ctypes.POINTER(ctypes.c_float)]
    L.dvqls_workspace_size.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp]
    L.dvqls_workspace_size.restype = ctypes.c_size_t
    L.dvqls_nccl_unique_id.argtypes = [vp]
    L.dvqls_build_info.restype = ctypes.c_char_p
    L.dvqls_shard_range.argtypes = [ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int64)]
    L.dvqls_cost_grad.argtypes = [vp, dp, dp, dp, dp]
    L.dvqls_cost_grad_dev.argtypes = [vp, vp, vp]
    L.dvqls_check.argtypes = [vp]
    L.dvqls_num_graphs.argtypes = [vp]
    for name in EXPORTED:
        if name not in ("dvqls_destroy", "dvqls_last_error", "dvqls_num_circuits", "dvqls_stream",
                        "dvqls_build_info", "dvqls_num_observables", "dvqls_decompose_error",
                        "dvqls_workspace_size"):
            getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _ptr(x):
    return ctypes.c_void_p(x.data_ptr() if hasattr(x, "data_ptr") else int(x))


def _check(rc, ctx=None):
    if rc == DVQLS_OK:
        return
    msg = load().dvqls_last_error(ctx).decode()
    if rc == DVQLS_E_DEGENERATE:
        raise DegenerateError(rc, msg)
    raise DvqlsError(rc, msg)


def dvqls_nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().dvqls_nccl_unique_id(buf))
    return buf.raw


def dvqls_shard_range(n_circuits: int, rank: int, world: int):
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(load().dvqls_shard_range(int(n_circuits), int(rank), int(world), ctypes.byref(a), ctypes.byref(b)))
    return int(a.value), int(b.value)


def dvqls_build_info() -> str:
    return load().dvqls_build_info().decode()


class Context:
    """Owns one dvqls_ctx*.  Methods mirror the C entry points."""

    def __init__(self, n, layers, paulis: bytes, coeffs, bkind=DVQLS_B_UNIFORM, b=None, device=-1, rank=0,
                 world=1, nccl_id: bytes | None = None, entangler=0, stream=None, timing=False, max_batch=16,
                 mode=0, workspace=None, **extra):
        """workspace: None (the library allocates its device tables once, here) or caller-owned device
        memory -- a CUDA torch tensor (kept alive by the context) or an (address, bytes) pair -- of at
        least workspace_size(...) bytes, 256-byte aligned (dvqls_opts.workspace_dev).
        extra: the remaining dvqls_opts fields by name (virtual_rank, virtual_world, allreduce,
        p2p_timeout_ms, host_allgather (a HOST_ALLGATHER, see make_host_allgather), graphs, pdl,
        stage, stream_grid, variant, prefix)."""
        L = load()
        self.n, self.layers = int(n), int(layers)
        self.P = 3 * self.n * self.layers
        self.L = len(paulis) // self.n
        if len(paulis) != self.L * self.n:
            raise ValueError("pauli_terms length must be n_terms * n")
        co = np.ascontiguousarray(coeffs, dtype=np.float64)
        if co.dtype != np.float64 or co.size != 2 * self.L:
            raise ValueError("coeffs must be 2*L interleaved doubles")
        self._keep = []
        bp = _BPrep(bkind, None)
        if bkind == DVQLS_B_AMPLITUDES:
            amps = np.ascontiguousarray(np.asarray(b, dtype=np.complex128)).view(np.float64).copy()
            self._keep.append(amps)
            bp.amps = _dp(amps)
        idbuf = None
        if nccl_id is not None:
            idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
            self._keep.append(idbuf)
        sp = None
        if stream is not None:
            sp = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        wp, wb = None, 0
        if workspace is not None:
            if hasattr(workspace, "data_ptr"):
                wp, wb = workspace.data_ptr(), workspace.numel() * workspace.element_size()
                self._keep.append(workspace)
            else:
                wp, wb = int(workspace[0]), int(workspace[1])
        if extra.get("host_allgather") is not None:
            self._keep.append(extra["host_allgather"])  # the callback must outlive the context
        op = _opts(device, rank, world, ctypes.cast(idbuf, ctypes.c_void_p) if idbuf is not None else None,
                   entangler, sp, timing, max_batch, mode, (wp, wb), **extra)
        h = ctypes.c_void_p()
        rc = L.dvqls_create(ctypes.byref(h), self.n, self.layers, self.L, paulis, _dp(co), ctypes.byref(bp),
                            ctypes.byref(op))
        _check(rc, None)
        self.h = h
        self.max_batch = max_batch
        # per-call host buffers of the cost entry points, allocated once (their addresses cached)
        self._th_buf = np.empty(max(1, max_batch) * self.P)
        self._c_buf = np.empty(max(1, max_batch))
        self._ep_buf = np.empty(4 * max(1, max_batch))
        self._th_addr = self._th_buf.ctypes.data
        self._c_addr = self._c_buf.ctypes.data
        self._ep_addr = self._ep_buf.ctypes.data

    # --- host-buffer entry points --------------------------------------------
    def terms(self, theta) -> np.ndarray:
        """All 2(n+1)L^2 terms (a virtual-rank context fills only its block; the rest stays NaN)."""
        th = self._theta(theta, 1)
        out = np.full(self.num_circuits(), np.nan, dtype=np.float64)
        _check(load().dvqls_terms(self.h, _dp(th), _dp(out)), self.h)
        return out

    def cost(self, theta, with_E_Psi=False):
        th = self._theta(theta, 1)
        self._th_buf[:self.P] = th
        rc = _lib.dvqls_cost(self.h, self._th_addr, self._c_addr, self._ep_addr)
        if rc:
            _check(rc, self.h)
        ep = self._ep_buf
        return (float(self._c_buf[0]), complex(ep[0], ep[1]), complex(ep[2], ep[3])) if with_E_Psi \
            else float(self._c_buf[0])

    def global_cost(self, theta, with_beta=False):
        """NEXT-3: (C_L, C_G, E, Psi[, beta]) of one theta (Eq. 1 and Alg. 1 forms)."""
        th = self._theta(theta, 1)
        o = np.empty(6)
        beta = np.empty(2 * self.L)
        _check(load().dvqls_global_cost(self.h, _dp(th), _dp(o), _dp(beta)), self.h)
        res = (float(o[0]), float(o[5]), complex(o[1], o[2]), complex(o[3], o[4]))
        return res + (beta[0::2] + 1j * beta[1::2],) if with_beta else res

    def costs_dev(self, K, thetas_dev, out6_dev, beta_dev=None):
        _check(load().dvqls_costs_dev(self.h, int(K), _ptr(thetas_dev), _ptr(out6_dev),
                                      _ptr(beta_dev) if beta_dev is not None else None), self.h)

    def cost_batch(self, thetas):
        th = np.ascontiguousarray(thetas, dtype=np.float64)
        K = th.shape[0]
        th = self._theta(th, K)
        if K > self.max_batch:  # the library rejects it: report through its error path
            _check(load().dvqls_cost_batch(self.h, K, th.ctypes.data, self._c_addr, self._ep_addr), self.h)
        self._th_buf[:K * self.P] = th
        rc = _lib.dvqls_cost_batch(self.h, K, self._th_addr, self._c_addr, self._ep_addr)
        if rc:
            _check(rc, self.h)
        return self._c_buf[:K].copy(), self._ep_buf[:4 * K].reshape(K, 4).copy()

    def cost_grad(self, theta, with_E_Psi=False):
        """Parameter-shift gradient (dvqls_cost_grad): (C, dC/dtheta[P]) [+ (E, Psi)]."""
        th = self._theta(theta, 1)
        c = np.empty(1)
        g = np.empty(self.P)
        ep = np.empty(4)
        _check(load().dvqls_cost_grad(self.h, _dp(th), _dp(c), _dp(g), _dp(ep)), self.h)
        if with_E_Psi:
            return float(c[0]), g, complex(ep[0], ep[1]), complex(ep[2], ep[3])
        return float(c[0]), g

    def cost_grad_dev(self, theta_dev, out_dev):
        _check(load().dvqls_cost_grad_dev(self.h, _ptr(theta_dev), _ptr(out_dev)), self.h)

    def check(self):
        """dvqls_check: synchronise and raise on an asynchronous failure (peer timeout)."""
        _check(load().dvqls_check(self.h), self.h)

    def num_graphs(self) -> int:
        return int(load().dvqls_num_graphs(self.h))

    def terms_subset(self, theta, idx) -> np.ndarray:
        th = self._theta(theta, 1)
        ix = np.ascontiguousarray(idx, dtype=np.int64)
        out = np.empty(ix.size, dtype=np.float64)
        _check(load().dvqls_terms_subset(self.h, _dp(th), ix.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                         ix.size, _dp(out)), self.h)
        return out

    def state(self, theta) -> np.ndarray:
        """|x(theta)> = V(theta)|0> from the GPU prefix kernel (Alg. 1 Step 5)."""
        th = self._theta(theta, 1)
        out = np.empty(2 << self.n, dtype=np.float64)
        _check(load().dvqls_state(self.h, _dp(th), _dp(out)), self.h)
        return out.view(np.complex128)

    # --- device-resident entry points (torch tensors or raw pointers) --------
    def cost_dev(self, K, thetas_dev, out_dev):
        _check(load().dvqls_cost_dev(self.h, int(K), _ptr(thetas_dev), _ptr(out_dev)), self.h)

    def terms_local_dev(self, theta_dev, out_dev):
        _check(load().dvqls_terms_local_dev(self.h, _ptr(theta_dev), _ptr(out_dev)), self.h)

    # --- introspection -----------------------------------------------------------
    def num_circuits(self) -> int:
        return int(load().dvqls_num_circuits(self.h))

    def local_range(self):
        a, b = ctypes.c_int64(), ctypes.c_int64()
        _check(load().dvqls_local_range(self.h, ctypes.byref(a), ctypes.byref(b)), self.h)
        return int(a.value), int(b.value)

    def stream_ptr(self) -> int:
        return int(load().dvqls_stream(self.h) or 0)

    def num_observables(self) -> int:
        return int(load().dvqls_num_observables(self.h))

    def grid(self) -> int:
        return int(load().dvqls_launch_grid(self.h))

    def launches_per_call(self) -> int:
        return int(load().dvqls_launches_per_call(self.h))

    def last_timings(self):
        ms = (ctypes.c_float * 4)()
        _check(load().dvqls_last_timings(self.h, ms), self.h)
        return {"prefix_ms": ms[0], "hadamard_ms": ms[1], "reduce_ms": ms[2], "call_ms": ms[3]}

    def destroy(self):
        if getattr(self, "h", None):
            load().dvqls_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def _theta(self, theta, K):
        th = np.ascontiguousarray(theta, dtype=np.float64).reshape(-1)
        if th.size != K * self.P:
            raise ValueError(f"theta must have K*P = {K}*{self.P} entries (P = 3 n d)")
        return th


# C-ABI-named functional wrappers --------------------------------------------------
def workspace_size(n_qubits, layers, n_terms, device=-1, rank=0, world=1, max_batch=16, mode=0, **extra) -> int:
    """dvqls_workspace_size: device bytes a context carves from a caller workspace (0 = invalid)."""
    op = _opts(device, rank, world, None, 0, None, False, max_batch, mode, **extra)
    return int(load().dvqls_workspace_size(int(n_qubits), int(layers), int(n_terms), ctypes.byref(op)))


def dvqls_create(n_qubits, layers, pauli_terms: bytes, coeffs, b_prep=(DVQLS_B_UNIFORM, None), **opts) -> Context:
    kind, amps = b_prep
    return Context(n_qubits, layers, pauli_terms, coeffs, kind, amps, **opts)


def dvqls_terms(ctx: Context, theta) -> np.ndarray:
    return ctx.terms(theta)


def dvqls_cost(ctx: Context, theta) -> float:
    return ctx.cost(theta)


def dvqls_cost_batch(ctx: Context, thetas):
    return ctx.cost_batch(thetas)[0]


def dvqls_destroy(ctx: Context) -> None:
    ctx.destroy()


def decompose(A, eps: float, max_terms: int = 4096, device: int = -1, timing: bool = False):
    """NEXT-4 on the GPU: pruned, ordered LCU [(c, pauli_string)] of a dense A, and ||c||_2
    (and the device milliseconds with timing=True)."""
    A = np.ascontiguousarray(A, dtype=np.complex128)
    N = A.shape[0]
    n = N.bit_length() - 1
    a = A.view(np.float64).reshape(-1)
    chars = ctypes.create_string_buffer(max_terms * n)
    co = np.empty(2 * max_terms)
    L, norm, ms = ctypes.c_int64(), ctypes.c_double(), ctypes.c_float()
    rc = load().dvqls_decompose(n, _dp(a), float(eps), max_terms, chars, _dp(co), ctypes.byref(L),
                                ctypes.byref(norm), device, ctypes.byref(ms) if timing else None)
    if rc:
        raise DvqlsError(rc, load().dvqls_decompose_error().decode())
    raw = chars.raw
    terms = [(complex(co[2 * i], co[2 * i + 1]), raw[i * n:(i + 1) * n].decode()) for i in range(L.value)]
    return (terms, norm.value, float(ms.value)) if timing else (terms, norm.value)


def pauli_coefficients(A, device: int = -1) -> np.ndarray:
    """NEXT-4: all 4^n coefficients as C[m, z] (x-mask m, z-mask z)."""
    A = np.ascontiguousarray(A, dtype=np.complex128)
    N = A.shape[0]
    n = N.bit_length() - 1
    out = np.empty(2 * N * N)
    rc = load().dvqls_pauli_coefficients(n, _dp(A.view(np.float64).reshape(-1)), _dp(out), device)
    if rc:
        raise DvqlsError(rc, load().dvqls_decompose_error().decode())
    return out.view(np.complex128).reshape(N, N)


def task_observable(n: int, pauli_l: str, pauli_k: str, s: int):
    """NEXT-2 host algebra (no device): (x_mask, z_mask, phase) of A_l X_j A_k / A_l A_k."""
    m, z, q = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_int()
    rc = load().dvqls_task_observable(n, pauli_l.encode(), pauli_k.encode(), s, ctypes.byref(m), ctypes.byref(z),
                                      ctypes.byref(q))
    if rc:
        raise DvqlsError(rc, "dvqls_task_observable")
    return int(m.value), int(z.value), int(q.value)


def from_workload(w, **opts) -> Context:
    """Context for a dvqls_inputs.configs.Workload."""
    chars, co = w.arrays()
    return Context(w.n, w.layers, chars, co, w.bkind, w.b, entangler=w.entangler, **opts)
