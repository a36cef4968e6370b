"""Python mirror of the reference's ``tve::Engine`` over the C ABI (include/tvegpu.h).

Same names, argument meaning and error behaviour as engine.hpp:83-143:
``Engine(problem)`` ~ ``Engine(mesh, pre, material, mech_bcs, thermal_bcs,
sources, config)``; ``step()`` raises :class:`InstabilityError` carrying
``step`` and ``node`` (errors.hpp:21-27); ``state()`` returns T, u, u_prev and
the viscous history in original numbering.  Every call goes through
``libtvegpu.so`` (hand-written sm_100a kernels); there is no CPU fallback — a
missing library or device raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import sys
import time

import numpy as np

from .problem import H8, Problem

_HERE = os.path.dirname(os.path.abspath(__file__))
# TVEGPU_LIB selects an experimental build variant (csrc/Makefile `variant` target).
_TIMING = bool(os.environ.get("TVEGPU_TIMING"))
_LIBPATH = os.environ.get("TVEGPU_LIB") or os.path.join(_HERE, "lib", "libtvegpu.so")
_LIB = None
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


# errors.hpp:8-33
class TveError(RuntimeError):
    status = 7


class ParseError(TveError):
    status = 1


class ValidationError(TveError):
    status = 2

    def __init__(self, msg, step=-1, element=-1):
        super().__init__(msg)
        self.step, self.element = step, element


class InstabilityError(TveError):
    status = 3

    def __init__(self, msg, step=-1, node=-1):
        super().__init__(msg)
        self.step, self.node = step, node


class IoError(TveError):
    status = 4


class CudaError(TveError):
    status = 5


class NcclError(TveError):
    status = 6


_BY_STATUS = {1: ParseError, 2: ValidationError, 3: InstabilityError, 4: IoError, 5: CudaError, 6: NcclError}


class COptions(C.Structure):
    _fields_ = [("device", C.c_int32), ("nranks", C.c_int32), ("rank", C.c_int32), ("nccl_unique_id", C.c_void_p),
                ("reorder", C.c_int32), ("diagnostics", C.c_int32), ("steps_per_graph", C.c_int32),
                ("halo_transport", C.c_int32), ("slot_fp32", C.c_int32)]


HALO_PEER, HALO_NCCL = 0, 1  # tvegpu.h TVEGPU_HALO_*


class CPlanView(C.Structure):
    _fields_ = [("nranks", C.c_int32), ("rank", C.c_int32), ("nn", C.c_int32), ("num_elements", C.c_int32),
                ("num_boundary_elements", C.c_int32), ("num_nodes", C.c_int32), ("element_orig", _ip),
                ("node_orig", _ip), ("conn", _ip), ("csr_offsets", _ip), ("csr_slots", _ip),
                ("num_neighbors", C.c_int32), ("neighbor_ranks", _ip), ("send_offsets", _ip), ("send_slots", _ip),
                ("recv_offsets", _ip), ("element_owner", _ip), ("num_elements_global", C.c_int32),
                ("num_chunks", C.c_int32), ("chunk_start", _ip), ("chunk_node_off", _ip), ("chunk_nodes", _ip),
                ("chunk_node_slot", C.POINTER(C.c_uint16)), ("chunk_conn", C.POINTER(C.c_uint16)),
                ("max_chunk_slots", C.c_int32)]


EXPORTS = {
    "tvegpu_abi_version": (C.c_int32, []),
    "tvegpu_status_string": (C.c_char_p, [C.c_int]),
    "tvegpu_create_error": (C.c_char_p, []),
    "tvegpu_default_options": (None, [C.c_void_p]),
    "tvegpu_create": (C.c_int, [C.c_void_p, C.c_void_p, C.POINTER(C.c_void_p)]),
    "tvegpu_destroy": (None, [C.c_void_p]),
    "tvegpu_step": (C.c_int, [C.c_void_p, C.c_int64]),
    "tvegpu_get_temperatures": (C.c_int, [C.c_void_p, _dp]),
    "tvegpu_get_displacements": (C.c_int, [C.c_void_p, _dp, _dp]),
    "tvegpu_get_viscous": (C.c_int, [C.c_void_p, _dp]),
    "tvegpu_make_snapshot": (C.c_int, [C.c_void_p, _dp, _dp]),
    "tvegpu_time": (C.c_double, [C.c_void_p]),
    "tvegpu_step_count": (C.c_int64, [C.c_void_p]),
    "tvegpu_set_state": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, C.c_double, C.c_int64]),
    "tvegpu_set_nodal_sources": (C.c_int, [C.c_void_p, _dp]),
    "tvegpu_step_io": (C.c_int, [C.c_void_p, _dp, C.c_int64, _dp, _dp]),
    "tvegpu_set_motion_override": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, _ip]),
    "tvegpu_get_summary": (C.c_int, [C.c_void_p, C.c_void_p]),
    "tvegpu_total_energy": (C.c_int, [C.c_void_p, _dp, _dp]),
    "tvegpu_load_mesh": (C.c_int, [C.c_char_p, C.c_uint64, C.POINTER(C.c_void_p), C.c_void_p]),
    "tvegpu_mesh_get_view": (None, [C.c_void_p, C.c_void_p]),
    "tvegpu_mesh_destroy": (None, [C.c_void_p]),
    "tvegpu_checkpoint_size": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "tvegpu_save_checkpoint": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "tvegpu_load_checkpoint": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "tvegpu_ablation_volume": (C.c_int, [C.c_void_p, C.c_double, C.c_int32, _dp, C.POINTER(C.c_int64)]),
    "tvegpu_element_fields": (C.c_int, [C.c_void_p, _dp, _dp]),
    "tvegpu_get_diagnostics": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "tvegpu_last_error": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int32)]),
    "tvegpu_critical_timestep": (C.c_int, [C.c_void_p, _dp, _dp]),
    "tvegpu_plan_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "tvegpu_plan_get": (C.c_int, [C.c_void_p, C.POINTER(CPlanView)]),
    "tvegpu_plan_destroy": (None, [C.c_void_p]),
    "tvegpu_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "tvegpu_peer_export": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]),
    "tvegpu_peer_attach": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.POINTER(C.c_size_t), C.c_int32]),
    "tvegpu_halo_peer": (C.c_int32, [C.c_void_p]),
    "tvegpu_peer_detach": (C.c_int, [C.c_void_p]),
    "tvegpu_peer_attach_solo": (C.c_int, [C.c_void_p]),
    "tvegpu_stream": (C.c_void_p, [C.c_void_p]),
    "tvegpu_kernels_per_step": (C.c_int32, [C.c_void_p]),
    "tvegpu_affine_chunks": (C.c_int32, [C.c_void_p]),
    "tvegpu_halo_info": (C.c_int, [C.c_void_p, _ip, C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "tvegpu_enqueue_steps": (C.c_int, [C.c_void_p, C.c_int64]),
    "tvegpu_sync": (C.c_int, [C.c_void_p]),
    "tvegpu_profile_kernels": (C.c_int, [C.c_void_p, C.c_int32, _dp, C.POINTER(C.c_int32), C.c_char_p,
                                         C.c_size_t]),
    "tvegpu_group_create": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.POINTER(C.c_void_p)]),
    "tvegpu_group_step": (C.c_int, [C.c_void_p, C.c_int64]),
    "tvegpu_group_get_fields": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
    "tvegpu_group_get_state": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp]),
    "tvegpu_group_set_state": (C.c_int, [C.c_void_p, _dp, _dp, _dp, _dp, C.c_double, C.c_int64]),
    "tvegpu_group_set_nodal_sources": (C.c_int, [C.c_void_p, _dp]),
    "tvegpu_group_step_io": (C.c_int, [C.c_void_p, _dp, C.c_int64, _dp, _dp]),
    "tvegpu_group_time": (C.c_double, [C.c_void_p]),
    "tvegpu_group_step_count": (C.c_int64, [C.c_void_p]),
    "tvegpu_group_last_error": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t, C.POINTER(C.c_int64),
                                          C.POINTER(C.c_int32)]),
    "tvegpu_group_checkpoint_size": (C.c_int, [C.c_void_p, C.POINTER(C.c_uint64)]),
    "tvegpu_group_save_checkpoint": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "tvegpu_group_load_checkpoint": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64]),
    "tvegpu_group_destroy": (None, [C.c_void_p]),
}


def build(force=False):
    """Compile csrc/ for sm_100a into lib/libtvegpu.so (nvcc cross-compiles without a GPU)."""
    cmd = ["make", "-s", "-C", os.path.join(_HERE, "csrc")]
    if force:
        subprocess.run(cmd + ["clean"], check=True)
    subprocess.run(cmd, check=True)


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(_LIBPATH):
            raise CudaError(f"{_LIBPATH} missing: run paper_2009_10400_b200.build() (no CPU fallback exists)")
        L = C.CDLL(_LIBPATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


# tvegpu_motion_fn: int32 (*)(void* user, int32 node, double t, double* disp)
MOTION_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_int32, C.c_double, _dp)


def motion_callback(fn):
    """Wraps fn(node, t) -> None or (dx, dy, dz) as a tvegpu_motion_fn (keep a reference)."""
    def cb(_user, node, t, out):
        v = fn(int(node), float(t))
        if v is None:
            return 0
        out[0], out[1], out[2] = float(v[0]), float(v[1]), float(v[2])
        return 1
    return MOTION_FN(cb)


class _Summary(C.Structure):
    _fields_ = [("steps", C.c_int64), ("time", C.c_double), ("max_temperature", C.c_double),
                ("min_disp", C.c_double * 3), ("max_disp", C.c_double * 3)]


def _P(a):
    return None if a is None else a.ctypes.data_as(_dp)


def _in(a, n, name):
    """An input array for the C side: float64, C-contiguous, exactly n values (a copy
    only when the caller's array is not already in that form)."""
    if a is None:
        return None
    v = np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
    if v.size != n:
        raise ValueError(f"{name}: expected {n} values, got {v.size}")
    return v


def _out(a, n, name):
    """A caller-supplied output buffer the C side writes n doubles into: it must be
    float64, C-contiguous and hold exactly n values (no silent copy: the caller
    expects the data in this very array)."""
    if a is None:
        return None
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags.c_contiguous or not a.flags.writeable:
        raise ValueError(f"{name}: expected a writeable C-contiguous float64 numpy array")
    if a.size != n:
        raise ValueError(f"{name}: expected {n} values, got {a.size}")
    return a


def critical_timestep(problem: Problem):
    """critical_timestep(mesh, material) (mesh.hpp:92-97) -> (thermal, mechanical)."""
    c, keep = problem.to_c()
    th, me = C.c_double(), C.c_double()
    rc = lib().tvegpu_critical_timestep(C.byref(c), C.byref(th), C.byref(me))
    if rc:
        raise _BY_STATUS.get(rc, TveError)(lib().tvegpu_create_error().decode())
    return th.value, me.value


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = lib().tvegpu_nccl_unique_id(buf)
    if rc:
        raise NcclError(lib().tvegpu_create_error().decode())
    return buf.raw


class _MeshView(C.Structure):
    _fields_ = [("kind", C.c_int32), ("num_nodes", C.c_int32), ("num_elements", C.c_int32),
                ("nodes", C.POINTER(C.c_double)), ("elements", C.POINTER(C.c_int32)),
                ("fiber_dirs", C.POINTER(C.c_double)), ("expansion_axes", C.POINTER(C.c_double)),
                ("num_node_sets", C.c_int32), ("node_set_names", C.POINTER(C.c_char_p)),
                ("node_set_offsets", C.POINTER(C.c_int32)), ("node_set_items", C.POINTER(C.c_int32)),
                ("num_element_sets", C.c_int32), ("element_set_names", C.POINTER(C.c_char_p)),
                ("element_set_offsets", C.POINTER(C.c_int32)), ("element_set_items", C.POINTER(C.c_int32))]


def load_mesh(src):
    """load_mesh / load_mesh_file (mesh.hpp:73-79): parse the SPEC.md:88 text format (str,
    bytes or a path) with the library's parallel parser.  Returns dict(kind, nodes (N,3),
    elements (E,nn) 0-based, fiber_dirs, expansion_axes, node_sets, element_sets)."""
    if isinstance(src, (bytes, bytearray)):
        data = bytes(src)
    elif isinstance(src, str) and ("\n" in src or src.lstrip().startswith("$")):
        data = src.encode()
    else:
        with open(src, "rb") as f:
            data = f.read()
    h, v = C.c_void_p(), _MeshView()
    rc = lib().tvegpu_load_mesh(data, len(data), C.byref(h), C.byref(v))
    if rc:
        raise _BY_STATUS.get(rc, TveError)(lib().tvegpu_create_error().decode())
    try:
        N, E = v.num_nodes, v.num_elements
        nn = 8 if v.kind == H8 else 4

        def arr(ptr, n, dt=np.float64):
            return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)

        def sets(n, names, off, items):
            out = {}
            if n:
                o = arr(off, n + 1, np.int32)
                it = arr(items, int(o[-1]), np.int32) if o[-1] else np.zeros(0, np.int32)
                for k in range(n):
                    out[names[k].decode()] = it[o[k]:o[k + 1]]
            return out
        return dict(kind=v.kind, nodes=arr(v.nodes, 3 * N).reshape(N, 3),
                    elements=arr(v.elements, nn * E, np.int32).reshape(E, nn),
                    fiber_dirs=arr(v.fiber_dirs, 3 * E).reshape(E, 3) if v.fiber_dirs else None,
                    expansion_axes=arr(v.expansion_axes, 6 * E).reshape(E, 6) if v.expansion_axes else None,
                    node_sets=sets(v.num_node_sets, v.node_set_names, v.node_set_offsets, v.node_set_items),
                    element_sets=sets(v.num_element_sets, v.element_set_names, v.element_set_offsets,
                                      v.element_set_items))
    finally:
        lib().tvegpu_mesh_destroy(h)


def plan(problem: Problem, nranks=1, rank=0, reorder=True):
    """The integer maps of one rank's layout (host-only; no GPU needed)."""
    c, keep = problem.to_c()
    h = C.c_void_p()
    rc = lib().tvegpu_plan_create(C.byref(c), nranks, rank, int(reorder), C.byref(h))
    if rc:
        raise _BY_STATUS.get(rc, TveError)(lib().tvegpu_create_error().decode())
    try:
        v = CPlanView()
        lib().tvegpu_plan_get(h, C.byref(v))

        def arr(ptr, n):
            return np.ctypeslib.as_array(ptr, shape=(n,)).copy() if n else np.zeros(0, np.int32)

        E, N, nn, nb = v.num_elements, v.num_nodes, v.nn, v.num_neighbors
        off = arr(v.csr_offsets, N + 1)
        send_off = arr(v.send_offsets, nb + 1)
        recv_off = arr(v.recv_offsets, nb + 1)
        return dict(nranks=v.nranks, rank=v.rank, nn=nn, num_elements=E, num_boundary_elements=v.num_boundary_elements,
                    num_nodes=N, element_orig=arr(v.element_orig, E), node_orig=arr(v.node_orig, N),
                    conn=arr(v.conn, E * nn).reshape(E, nn), csr_offsets=off, csr_slots=arr(v.csr_slots, int(off[-1])),
                    neighbors=arr(v.neighbor_ranks, nb), send_offsets=send_off,
                    send_slots=arr(v.send_slots, int(send_off[-1])), recv_offsets=recv_off,
                    element_owner=arr(v.element_owner, v.num_elements_global),
                    chunk_start=arr(v.chunk_start, v.num_chunks + 1),
                    chunk_node_off=arr(v.chunk_node_off, v.num_chunks + 1),
                    chunk_nodes=arr(v.chunk_nodes, int(arr(v.chunk_node_off, v.num_chunks + 1)[-1])),
                    chunk_node_slot=arr(v.chunk_node_slot, int(arr(v.chunk_node_off, v.num_chunks + 1)[-1])),
                    chunk_conn=arr(v.chunk_conn, E * nn).reshape(E, nn), max_chunk_slots=v.max_chunk_slots)
    finally:
        lib().tvegpu_plan_destroy(h)


class PartitionGroup:
    """nparts RCB partitions of one problem stepped together on one GPU by the
    multi-GPU step code (tvegpu_group_*): the same calls as :class:`Engine`.
    halo_transport: HALO_PEER (default; the peer-memory send kernels, with the other
    partitions' buffers standing in for the other GPUs) or HALO_NCCL (pack + exchange,
    device copies instead of ncclSend/ncclRecv)."""

    def __init__(self, problem: Problem, nparts: int, *, device: int = -1, steps_per_graph: int = 64,
                 halo_transport: int = HALO_PEER, slot_fp32: bool = False):
        L = lib()
        self.problem = problem
        self._c, self._keep = problem.to_c()
        o = COptions()
        L.tvegpu_default_options(C.byref(o))
        o.device = device
        o.steps_per_graph = steps_per_graph
        o.halo_transport = halo_transport
        o.slot_fp32 = int(slot_fp32)
        h = C.c_void_p()
        rc = L.tvegpu_group_create(C.byref(self._c), nparts, C.byref(o), C.byref(h))
        if rc:
            raise _BY_STATUS.get(rc, TveError)(L.tvegpu_create_error().decode())
        self._h = h
        self.N, self.E, self.P = problem.num_nodes, problem.num_elements, problem.prony_count

    def close(self):
        if getattr(self, "_h", None):
            lib().tvegpu_group_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, rc):
        msg = C.create_string_buffer(512)
        st, nd = C.c_int64(-1), C.c_int32(-1)
        lib().tvegpu_group_last_error(self._h, msg, 512, C.byref(st), C.byref(nd))
        text = msg.value.decode()
        if rc == 3:
            raise InstabilityError(text, st.value, nd.value)
        if rc == 2:
            raise ValidationError(text, st.value, nd.value)
        raise _BY_STATUS.get(rc, TveError)(text)

    def step(self, n: int = 1):
        rc = lib().tvegpu_group_step(self._h, n)
        if rc:
            self._raise(rc)

    def time(self) -> float:
        return lib().tvegpu_group_time(self._h)

    def step_count(self) -> int:
        return lib().tvegpu_group_step_count(self._h)

    def state(self):
        T = np.full(self.N, np.nan)
        u = np.full(3 * self.N, np.nan)
        up = np.full(3 * self.N, np.nan)
        th = np.full(9 * self.E * self.P, np.nan)
        rc = lib().tvegpu_group_get_state(self._h, _P(T), _P(u), _P(up), _P(th) if th.size else None)
        if rc:
            self._raise(rc)
        return dict(T=T, u=u, u_prev=up, viscous=th, time=self.time(), step=self.step_count())

    def fields(self):
        s = self.state()
        return dict(T=s["T"], u=s["u"], viscous=s["viscous"])

    def set_state(self, T=None, u=None, u_prev=None, viscous=None, time=0.0, step=0):
        arrs = [_in(T, self.N, "T"), _in(u, 3 * self.N, "u"), _in(u_prev, 3 * self.N, "u_prev"),
                _in(viscous, 9 * self.E * self.P, "viscous")]
        rc = lib().tvegpu_group_set_state(self._h, *(_P(a) for a in arrs), time, step)
        if rc:
            self._raise(rc)

    def set_nodal_sources(self, power):
        self._src = _in(power, self.N, "power")
        rc = lib().tvegpu_group_set_nodal_sources(self._h, _P(self._src))
        if rc:
            self._raise(rc)

    def step_io(self, power=None, n=1, T=None, u=None):
        src = _in(power, self.N, "power")
        rc = lib().tvegpu_group_step_io(self._h, _P(src), int(n), _P(_out(T, self.N, "T")),
                                        _P(_out(u, 3 * self.N, "u")))
        if rc:
            self._raise(rc)
        return T, u

    def save_checkpoint(self) -> bytes:
        n = C.c_uint64()
        rc = lib().tvegpu_group_checkpoint_size(self._h, C.byref(n))
        if rc:
            self._raise(rc)
        buf = C.create_string_buffer(n.value)
        rc = lib().tvegpu_group_save_checkpoint(self._h, buf, n.value)
        if rc:
            self._raise(rc)
        return buf.raw

    def load_checkpoint(self, data):
        rc = lib().tvegpu_group_load_checkpoint(self._h, bytes(data), len(data))
        if rc:
            self._raise(rc)


class Engine:
    """tve::Engine on a B200 (engine.hpp:83-143)."""

    def __init__(self, problem: Problem, *, device: int = -1, nranks: int = 1, rank: int = 0,
                 nccl_id: bytes | None = None, reorder: bool = True, diagnostics: bool = False,
                 steps_per_graph: int = 64, halo_transport: int = HALO_PEER, slot_fp32: bool = False):
        L = lib()
        self.problem = problem
        t0 = time.perf_counter()
        self._c, self._keep = problem.to_c()
        if _TIMING:
            print(f"[tvegpu setup] {'python problem -> C structs':28s} {1e3 * (time.perf_counter() - t0):8.1f} ms",
                  file=sys.stderr)
        o = COptions()
        L.tvegpu_default_options(C.byref(o))
        o.device, o.nranks, o.rank = device, nranks, rank
        self._id = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        o.nccl_unique_id = C.cast(self._id, C.c_void_p) if self._id is not None else None
        o.reorder, o.diagnostics, o.steps_per_graph = int(reorder), int(diagnostics), steps_per_graph
        o.halo_transport = halo_transport
        o.slot_fp32 = int(slot_fp32)
        self._opt = o
        h = C.c_void_p()
        t0 = time.perf_counter()
        rc = L.tvegpu_create(C.byref(self._c), C.byref(o), C.byref(h))
        if rc:
            raise _BY_STATUS.get(rc, TveError)(L.tvegpu_create_error().decode())
        if _TIMING:
            print(f"[tvegpu setup] {'tvegpu_create (total)':28s} {1e3 * (time.perf_counter() - t0):8.1f} ms",
                  file=sys.stderr)
        self._h = h
        self.N, self.E, self.P = problem.num_nodes, problem.num_elements, problem.prony_count

    def close(self):
        if getattr(self, "_h", None):
            lib().tvegpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _raise(self, rc):
        msg = C.create_string_buffer(512)
        st, nd = C.c_int64(-1), C.c_int32(-1)
        lib().tvegpu_last_error(self._h, msg, 512, C.byref(st), C.byref(nd))
        text = msg.value.decode()
        if rc == 3:
            raise InstabilityError(text, st.value, nd.value)
        if rc == 2:
            raise ValidationError(text, st.value, nd.value)
        raise _BY_STATUS.get(rc, TveError)(text)

    # ---- engine.hpp:89-97
    def step(self, n: int = 1):
        rc = lib().tvegpu_step(self._h, n)
        if rc:
            self._raise(rc)

    def enqueue(self, n: int):
        rc = lib().tvegpu_enqueue_steps(self._h, n)
        if rc:
            self._raise(rc)

    def sync(self):
        rc = lib().tvegpu_sync(self._h)
        if rc:
            self._raise(rc)

    def time(self) -> float:
        return lib().tvegpu_time(self._h)

    def step_count(self) -> int:
        return lib().tvegpu_step_count(self._h)

    def temperatures(self, out=None):
        T = np.empty(self.N) if out is None else _out(out, self.N, "out")
        rc = lib().tvegpu_get_temperatures(self._h, _P(T))
        if rc:
            self._raise(rc)
        return T

    def displacements(self, out=None, out_prev=None):
        u = np.empty(3 * self.N) if out is None else _out(out, 3 * self.N, "out")
        rc = lib().tvegpu_get_displacements(self._h, _P(u), _P(_out(out_prev, 3 * self.N, "out_prev")))
        if rc:
            self._raise(rc)
        return u

    # ---- engine.hpp:92 run(sink) -> RunSummary
    def run(self, sink=None, snapshot_interval=0.0, ablation_threshold=60.0, element_fields=False):
        """Advance problem.duration / dt steps; call sink(snapshot dict) every snapshot_interval
        (and at the end); return the RunSummary (engine.hpp:57-66) with per-step wall-time
        median / IQR measured over the chunks between snapshots."""
        import time as _time
        dt = self.problem.dt
        total = max(1, int(round(self.problem.duration / dt)))
        every = max(1, int(round(snapshot_interval / dt))) if snapshot_interval > 0 else total
        per, done = [], 0
        while done < total:
            k = min(every, total - done)
            t0 = _time.perf_counter()
            self.step(k)
            per.append((_time.perf_counter() - t0) / k)
            done += k
            if sink is not None and (snapshot_interval > 0 or done == total):
                T, u = self.make_snapshot()
                snap = dict(time=self.time(), step=self.step_count(), temperatures=T, displacements=u)
                if element_fields:
                    snap["det_f"], snap["max_principal_stress"] = self.element_fields()
                sink(snap)
        s = self.summary()
        per = np.sort(np.array(per))
        return dict(steps=s["steps"], final_time=s["time"], max_temperature=s["max_temperature"],
                    min_displacement=s["min_disp"], max_displacement=s["max_disp"],
                    ablation_volume=self.ablation_volume(ablation_threshold)[0] if ablation_threshold > 0 else 0.0,
                    median_step_seconds=float(per[len(per) // 2]),
                    iqr_step_seconds=float(per[(3 * len(per)) // 4] - per[len(per) // 4]))

    # ---- checkpoint / restart (engine.hpp:110-111)
    def save_checkpoint(self, path=None) -> bytes:
        """Versioned binary state image (original numbering); written to `path` if given."""
        n = C.c_uint64()
        rc = lib().tvegpu_checkpoint_size(self._h, C.byref(n))
        if rc:
            self._raise(rc)
        buf = C.create_string_buffer(n.value)
        rc = lib().tvegpu_save_checkpoint(self._h, buf, n.value)
        if rc:
            self._raise(rc)
        data = buf.raw
        if path is not None:
            with open(path, "wb") as f:
                f.write(data)
        return data

    def load_checkpoint(self, src):
        """Restore from bytes or a file path written by save_checkpoint (any partitioning)."""
        data = src if isinstance(src, (bytes, bytearray)) else open(src, "rb").read()
        rc = lib().tvegpu_load_checkpoint(self._h, bytes(data), len(data))
        if rc:
            self._raise(rc)

    # ---- run-level outputs on the device (engine.hpp:57-66)
    def summary(self):
        """RunSummary extrema: dict(steps, time, max_temperature, min_disp, max_disp)."""
        out = _Summary()
        rc = lib().tvegpu_get_summary(self._h, C.byref(out))
        if rc:
            self._raise(rc)
        return dict(steps=out.steps, time=out.time, max_temperature=out.max_temperature,
                    min_disp=np.array(out.min_disp[:]), max_disp=np.array(out.max_disp[:]))

    def total_energy(self, split=False):
        """total_energy (engine.hpp:108): kinetic + strain energy [J] ((kinetic, strain) if split)."""
        k, e = np.empty(1), np.empty(1)
        rc = lib().tvegpu_total_energy(self._h, _P(k), _P(e))
        if rc:
            self._raise(rc)
        return (float(k[0]), float(e[0])) if split else float(k[0] + e[0])

    def ablation_volume(self, threshold=60.0, deformed=True):
        """(volume [m^3], elements_above) of {T >= threshold} by exact tet clipping."""
        v, n = np.empty(1), C.c_int64()
        rc = lib().tvegpu_ablation_volume(self._h, float(threshold), 1 if deformed else 0, _P(v), C.byref(n))
        if rc:
            self._raise(rc)
        return float(v[0]), int(n.value)

    def element_fields(self):
        """(det F, max principal S_tilde) per element of the last mechanics phase (diagnostics=True)."""
        d, s = np.empty(self.E), np.empty(self.E)
        rc = lib().tvegpu_element_fields(self._h, _P(d), _P(s))
        if rc:
            self._raise(rc)
        return d, s

    def step_io(self, power=None, n=1, T=None, u=None):
        """set_nodal_sources(power) + step(n) + make_snapshot(T, u) in one call, the
        host copies overlapped with the step (tvegpu_step_io).  T/u are filled in place."""
        src = _in(power, self.N, "power")
        rc = lib().tvegpu_step_io(self._h, _P(src), int(n), _P(_out(T, self.N, "T")), _P(_out(u, 3 * self.N, "u")))
        if power is not None:
            self._src = src
        if rc:
            self._raise(rc)
        return T, u

    def make_snapshot(self, T=None, u=None):
        """Engine::make_snapshot (engine.hpp:99): T and u in one device read."""
        T = np.empty(self.N) if T is None else _out(T, self.N, "T")
        u = np.empty(3 * self.N) if u is None else _out(u, 3 * self.N, "u")
        rc = lib().tvegpu_make_snapshot(self._h, _P(T), _P(u))
        if rc:
            self._raise(rc)
        return T, u

    def state(self):
        T = self.temperatures()
        u = np.empty(3 * self.N)
        up = np.empty(3 * self.N)
        self.displacements(u, up)
        th = np.empty(9 * self.E * self.P)
        if th.size:
            rc = lib().tvegpu_get_viscous(self._h, _P(th))
            if rc:
                self._raise(rc)
        return dict(T=T, u=u, u_prev=up, viscous=th, time=self.time(), step=self.step_count())

    def set_state(self, T=None, u=None, u_prev=None, viscous=None, time=0.0, step=0):
        arrs = [_in(T, self.N, "T"), _in(u, 3 * self.N, "u"), _in(u_prev, 3 * self.N, "u_prev"),
                _in(viscous, 9 * self.E * self.P, "viscous")]
        rc = lib().tvegpu_set_state(self._h, *(_P(a) for a in arrs), time, step)
        if rc:
            self._raise(rc)

    def set_nodal_sources(self, power):
        self._src = _in(power, self.N, "power")
        rc = lib().tvegpu_set_nodal_sources(self._h, _P(self._src))
        if rc:
            self._raise(rc)

    # ---- MechBCs::motion_override (mechanics.hpp:43-46)
    def set_motion_override(self, fn, nodes=None):
        """fn(node, t) -> None or (dx, dy, dz): pins original node `node` at time t, applied
        after the fixed / prescribed components of every step (slow path: one host
        evaluation per candidate node and step).  nodes limits the candidates (default:
        every node, as the reference evaluates it).  fn = None removes it."""
        self._motion = None if fn is None else motion_callback(fn)
        ids = None if nodes is None else np.ascontiguousarray(nodes, dtype=np.int32).reshape(-1)
        self._motion_nodes = ids
        rc = lib().tvegpu_set_motion_override(self._h, C.cast(self._motion, C.c_void_p) if fn is not None else None,
                                              None, 0 if ids is None else ids.size,
                                              None if ids is None else ids.ctypes.data_as(_ip))
        if rc:
            self._raise(rc)

    # ---- engine.hpp:101-105
    def diagnostics(self):
        f = np.empty(3 * self.N)
        F = np.empty(9 * self.E)
        S = np.empty(9 * self.E)
        rc = lib().tvegpu_get_diagnostics(self._h, _P(f), _P(F), _P(S))
        if rc:
            self._raise(rc)
        return dict(f_int=f, F=F, S=S)

    # ---- measurement hooks
    @property
    def stream(self) -> int:
        return lib().tvegpu_stream(self._h) or 0

    def kernels_per_step(self) -> int:
        return lib().tvegpu_kernels_per_step(self._h)

    def affine_chunks(self) -> int:
        """H8: chunks whose elements are all affine (K3's short hourglass branch)."""
        return lib().tvegpu_affine_chunks(self._h)

    def peer_export(self) -> bytes:
        """This partition's peer-memory halo descriptor (tvegpu_peer_export): all-gather
        them over the ranks, then :meth:`peer_attach` on every rank."""
        n = C.c_size_t()
        rc = lib().tvegpu_peer_export(self._h, None, 0, C.byref(n))
        if rc:
            self._raise(rc)
        buf = C.create_string_buffer(n.value)
        rc = lib().tvegpu_peer_export(self._h, buf, n.value, C.byref(n))
        if rc:
            self._raise(rc)
        return buf.raw[:n.value]

    def peer_attach(self, blobs):
        """Attach the neighbours' descriptors (a list indexed by rank): the halo then moves
        by peer-memory stores from the boundary element kernels (tvegpu_peer_attach)."""
        bufs = [C.create_string_buffer(b, len(b)) for b in blobs]
        ptrs = (C.c_void_p * len(bufs))(*[C.cast(b, C.c_void_p) for b in bufs])
        lens = (C.c_size_t * len(bufs))(*[len(b) for b in blobs])
        rc = lib().tvegpu_peer_attach(self._h, ptrs, lens, len(bufs))
        if rc:
            self._raise(rc)

    def peer_attach_solo(self):
        """Measurement hook (tvegpu_peer_attach_solo): step this partition alone, halo stores
        into scratch, waits passing — for timing one rank of a P-GPU run on one device."""
        rc = lib().tvegpu_peer_attach_solo(self._h)
        if rc:
            self._raise(rc)

    def peer_detach(self):
        """Back to the NCCL halo (every rank must use the same transport)."""
        rc = lib().tvegpu_peer_detach(self._h)
        if rc:
            self._raise(rc)

    @property
    def halo_peer(self) -> bool:
        return bool(lib().tvegpu_halo_peer(self._h))

    def halo_info(self):
        """(neighbours, bytes sent, bytes received) per step of this partition's halo exchange."""
        nb, sb, rb = C.c_int32(), C.c_int64(), C.c_int64()
        rc = lib().tvegpu_halo_info(self._h, C.byref(nb), C.byref(sb), C.byref(rb))
        if rc:
            self._raise(rc)
        return nb.value, sb.value, rb.value

    def profile_kernels(self, nsteps: int):
        ms = np.zeros(8)
        cnt = C.c_int32(0)
        names = C.create_string_buffer(512)
        rc = lib().tvegpu_profile_kernels(self._h, nsteps, _P(ms), C.byref(cnt), names, 512)
        if rc:
            self._raise(rc)
        return dict(zip(names.value.decode().split(";"), ms[:cnt.value].tolist()))
