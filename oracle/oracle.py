"""ctypes wrapper of the CPU oracle (oracle/liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package.
The oracle is a fresh fp64 restatement of the reference API (tve_oracle.hpp);
it is pinned against SPEC.md's golden examples (tests/test_oracle_golden.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            build()
        L = C.CDLL(path)
        L.oracle_error.restype = C.c_char_p
        L.oracle_create.restype = C.c_void_p
        L.oracle_create.argtypes = [C.c_void_p]
        L.oracle_create_motion.restype = C.c_void_p
        L.oracle_create_motion.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_destroy.argtypes = [C.c_void_p]
        L.oracle_step.argtypes = [C.c_void_p, C.c_long, C.POINTER(C.c_long), C.POINTER(C.c_int)]
        L.oracle_get_state.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        L.oracle_set_state.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, C.c_double, C.c_long]
        L.oracle_time.restype = C.c_double
        L.oracle_time.argtypes = [C.c_void_p]
        L.oracle_step_count.restype = C.c_long
        L.oracle_step_count.argtypes = [C.c_void_p]
        L.oracle_set_nodal_sources.argtypes = [C.c_void_p, _dp]
        L.oracle_get_diagnostics.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp]
        L.oracle_total_energy.restype = C.c_double
        L.oracle_total_energy.argtypes = [C.c_void_p]
        L.oracle_precompute.argtypes = [C.c_void_p] + [_dp] * 7 + [_ip] * 3
        L.oracle_critical_timestep.argtypes = [C.c_void_p, _dp]
        L.oracle_ablation_volume.argtypes = [C.c_int, C.c_int, C.c_int, _dp, _ip, _dp, _dp, C.c_double, _dp,
                                             C.POINTER(C.c_long)]
        L.oracle_strain_energy.argtypes = [_dp, C.c_double, C.c_double, C.c_double, _dp, _dp]
        L.oracle_pk2_stress.argtypes = [_dp, C.c_double, C.c_double, C.c_double, _dp, _dp]
        L.oracle_total_pk2_stress.argtypes = [_dp, _dp, C.c_double, C.c_double, C.c_double, _dp, _dp]
        L.oracle_thermal_deformation_gradient.argtypes = [C.c_double, C.c_int] + [C.c_double] * 4 + [_dp] * 3
        L.oracle_prony_update.argtypes = [_dp, _dp, C.c_int, _dp, _dp, C.c_double, _dp]
        L.oracle_relaxation_function.argtypes = [C.c_double, C.c_int, _dp, _dp, _dp]
        L.oracle_interp_property.argtypes = [C.c_int, _dp, _dp, C.c_double, _dp]
        L.oracle_deformation_gradient.argtypes = [C.c_int, _dp, _dp, _dp]
        L.oracle_element_thermal_load.argtypes = [C.c_int, _dp, _dp, _dp, _dp, C.c_double, _dp]
        L.oracle_element_internal_force.argtypes = ([C.c_int, _dp, _dp, C.c_double, C.c_double, C.c_double, _dp,
                                                     _dp, _dp, C.c_int, _dp, _dp, C.c_double, C.c_double, _dp])
        L.oracle_hourglass_force.argtypes = [_dp, _dp, C.c_double, _dp]
        L.oracle_hourglass_basis.argtypes = [_dp, _dp, _dp]
        L.oracle_step_displacement.argtypes = [C.c_int, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double]
        L.oracle_step_temperature.argtypes = ([C.c_int, _dp, _dp, _dp, _dp, C.c_double, C.c_int, _dp, _dp]
                                              + [C.c_double] * 5 + [C.c_int])
        _LIB = L
    return _LIB


def P(a):
    """float64 pointer of a contiguous array (or None)."""
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def IP(a):
    if a is None:
        return None
    assert a.dtype == np.int32 and a.flags.c_contiguous
    return a.ctypes.data_as(_ip)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


class OracleError(RuntimeError):
    def __init__(self, status, msg, step=-1, node=-1):
        super().__init__(msg)
        self.status, self.step, self.node = status, step, node


class OracleEngine:
    """tve::Engine restated on the CPU (engine.hpp:83-143)."""

    def __init__(self, problem, workers=0, motion_override=None):
        """motion_override: fn(node, t) -> None or (dx, dy, dz) (MechBCs::motion_override,
        mechanics.hpp:43-46), evaluated for every node at t + dt of each step."""
        self.problem = problem
        self._c, self._keep = problem.to_c()
        self._c.workers = workers
        L = lib()
        if motion_override is not None:
            def cb(_user, node, t, out):
                v = motion_override(int(node), float(t))
                if v is None:
                    return 0
                out[0], out[1], out[2] = float(v[0]), float(v[1]), float(v[2])
                return 1
            self._motion = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_double, _dp)(cb)
            self._h = L.oracle_create_motion(C.byref(self._c), C.cast(self._motion, C.c_void_p), None)
        else:
            self._h = L.oracle_create(C.byref(self._c))
        if not self._h:
            raise OracleError(2, L.oracle_error().decode())
        self.N, self.E, self.P = problem.num_nodes, problem.num_elements, problem.prony_count

    def __del__(self):
        if getattr(self, "_h", None):
            try:
                lib().oracle_destroy(self._h)
            except TypeError:  # interpreter shutdown: module globals already cleared
                pass
            self._h = None

    def step(self, n=1):
        s, nd = C.c_long(-1), C.c_int(-1)
        rc = lib().oracle_step(self._h, n, C.byref(s), C.byref(nd))
        if rc:
            raise OracleError(rc, lib().oracle_error().decode(), s.value, nd.value)

    def state(self):
        T = np.empty(self.N)
        u = np.empty(3 * self.N)
        up = np.empty(3 * self.N)
        th = np.empty(9 * self.E * self.P)
        lib().oracle_get_state(self._h, P(T), P(u), P(up), P(th) if th.size else None)
        return dict(T=T, u=u, u_prev=up, viscous=th, time=self.time(), step=self.step_count())

    def set_state(self, T=None, u=None, u_prev=None, viscous=None, time=0.0, step=0):
        lib().oracle_set_state(self._h, P(f64(T)) if T is not None else None,
                               P(f64(u)) if u is not None else None,
                               P(f64(u_prev)) if u_prev is not None else None,
                               P(f64(viscous)) if viscous is not None else None, time, step)

    def set_nodal_sources(self, power):
        self._src = None if power is None else f64(power)
        lib().oracle_set_nodal_sources(self._h, P(self._src))

    def time(self):
        return lib().oracle_time(self._h)

    def step_count(self):
        return lib().oracle_step_count(self._h)

    def diagnostics(self):
        nn = self.problem.nn
        out = dict(f_int=np.empty(3 * self.N), F=np.empty(9 * self.E), S=np.empty(9 * self.E),
                   thermal_loads=np.empty(nn * self.E), forces=np.empty(3 * nn * self.E),
                   nodal_sources=np.empty(self.N))
        lib().oracle_get_diagnostics(self._h, *(P(out[k]) for k in
                                                ("f_int", "F", "S", "thermal_loads", "forces", "nodal_sources")))
        return out

    def total_energy(self):
        return lib().oracle_total_energy(self._h)


def precompute(problem):
    """Reference-layout precompute arrays (mesh.hpp:45-71)."""
    c, keep = problem.to_c()
    E, N, nn = problem.num_elements, problem.num_nodes, problem.nn
    out = dict(grads=np.empty(3 * nn * E), ref_volume=np.empty(E), det_jacobian=np.empty(E),
               lumped_mass=np.empty(N), heat_capacity_ref=np.empty(N), node_volume=np.empty(N),
               hourglass=np.empty(32 * E), adj_offsets=np.empty(N + 1, np.int32),
               adj_elem=np.empty(nn * E, np.int32), adj_local=np.empty(nn * E, np.int32))
    rc = lib().oracle_precompute(C.byref(c), *(P(out[k]) for k in ("grads", "ref_volume", "det_jacobian",
                                                                   "lumped_mass", "heat_capacity_ref",
                                                                   "node_volume", "hourglass")),
                                 *(IP(out[k]) for k in ("adj_offsets", "adj_elem", "adj_local")))
    if rc:
        raise OracleError(rc, lib().oracle_error().decode())
    return out


def critical_timestep(problem):
    c, keep = problem.to_c()
    out = np.empty(2)
    rc = lib().oracle_critical_timestep(C.byref(c), P(out))
    if rc:
        raise OracleError(rc, lib().oracle_error().decode())
    return float(out[0]), float(out[1])


def ablation_volume(kind, nodes, elements, T, threshold, disp=None):
    """ablation_volume -> (volume [m^3], elements_above); kind 'T4'/'H8' or 0/1."""
    k = 1 if kind in (1, "H8") else 0
    nodes = f64(np.asarray(nodes).reshape(-1))
    elements = np.ascontiguousarray(np.asarray(elements).reshape(-1), dtype=np.int32)
    T = f64(T)
    disp = None if disp is None else f64(np.asarray(disp).reshape(-1))
    vol, cnt = np.empty(1), C.c_long()
    nn = 8 if k else 4
    _chk(lib().oracle_ablation_volume(k, len(T), len(elements) // nn, P(nodes), IP(elements), P(T), P(disp),
                                      float(threshold), P(vol), C.byref(cnt)))
    return float(vol[0]), int(cnt.value)


def _chk(rc):
    if rc:
        raise OracleError(rc, lib().oracle_error().decode())


def strain_energy(Cm, mu, kappa, eta=0.0, fiber=None):
    out = np.empty(1)
    _chk(lib().oracle_strain_energy(P(f64(Cm).reshape(9)), mu, kappa, eta,
                                    P(f64(fiber)) if fiber is not None else None, P(out)))
    return float(out[0])


def pk2_stress(Cm, mu, kappa, eta=0.0, fiber=None):
    out = np.empty(9)
    _chk(lib().oracle_pk2_stress(P(f64(Cm).reshape(9)), mu, kappa, eta,
                                 P(f64(fiber)) if fiber is not None else None, P(out)))
    return out.reshape(3, 3)


def total_pk2_stress(F, Fth, mu, kappa, eta=0.0, fiber=None):
    out = np.empty(9)
    _chk(lib().oracle_total_pk2_stress(P(f64(F).reshape(9)), P(f64(Fth).reshape(9)), mu, kappa, eta,
                                       P(f64(fiber)) if fiber is not None else None, P(out)))
    return out.reshape(3, 3)


def thermal_deformation_gradient(T, kind, alpha_i, alpha_m=0.0, alpha_n=0.0, Tref=37.0,
                                 m=(1, 0, 0), n=(0, 1, 0)):
    out = np.empty(9)
    _chk(lib().oracle_thermal_deformation_gradient(T, kind, alpha_i, alpha_m, alpha_n, Tref,
                                                   P(f64(m)), P(f64(n)), P(out)))
    return out.reshape(3, 3)


def prony_update(S, hist, phi, tau, dt):
    h = f64(hist).reshape(-1).copy()
    out = np.empty(9)
    _chk(lib().oracle_prony_update(P(f64(S).reshape(9)), P(h), len(phi), P(f64(phi)), P(f64(tau)), dt, P(out)))
    return out.reshape(3, 3), h.reshape(-1, 3, 3)


def relaxation_function(t, phi, tau):
    out = np.empty(1)
    _chk(lib().oracle_relaxation_function(t, len(phi), P(f64(phi)), P(f64(tau)), P(out)))
    return float(out[0])


def interp_property(table, T):
    out = np.empty(1)
    _chk(lib().oracle_interp_property(len(table), P(f64([a for a, _ in table])), P(f64([b for _, b in table])),
                                      T, P(out)))
    return float(out[0])


def deformation_gradient(U, G):
    """U, G: (nn, 3) (column a of the 3 x nn matrices)."""
    out = np.empty(9)
    _chk(lib().oracle_deformation_gradient(U.shape[0], P(f64(U).reshape(-1)), P(f64(G).reshape(-1)), P(out)))
    return out.reshape(3, 3)


def element_thermal_load(F, G, D, Te, V):
    nn = G.shape[0]
    out = np.empty(nn)
    _chk(lib().oracle_element_thermal_load(nn, P(f64(F).reshape(9)), P(f64(G).reshape(-1)), P(f64(D).reshape(9)),
                                           P(f64(Te)), V, P(out)))
    return out


def element_internal_force(F, G, mu, kappa, eta, fiber, Fth, hist, phi, tau, dt, V):
    nn = G.shape[0]
    out = np.empty(3 * nn)
    h = f64(hist).reshape(-1).copy()
    _chk(lib().oracle_element_internal_force(nn, P(f64(F).reshape(9)), P(f64(G).reshape(-1)), mu, kappa, eta,
                                             P(f64(fiber)) if fiber is not None else None,
                                             P(f64(Fth).reshape(9)), P(h) if h.size else None, len(phi),
                                             P(f64(phi)) if len(phi) else None,
                                             P(f64(tau)) if len(phi) else None, dt, V, P(out)))
    return out.reshape(nn, 3), h.reshape(-1, 3, 3)


def hourglass_basis(X, G):
    out = np.empty(32)
    lib().oracle_hourglass_basis(P(f64(X).reshape(-1)), P(f64(G).reshape(-1)), P(out))
    return out.reshape(4, 8)


def hourglass_force(U, gamma, k):
    out = np.empty(24)
    lib().oracle_hourglass_force(P(f64(U).reshape(-1)), P(f64(gamma).reshape(-1)), k, P(out))
    return out.reshape(8, 3)


def step_displacement(u, uprev, f, M, R, gamma, dt):
    u, up = f64(u).copy(), f64(uprev).copy()
    N = M.size
    _chk(lib().oracle_step_displacement(N, P(u), P(up), P(f64(f)), P(f64(M)), P(f64(R)) if R is not None else None,
                                        gamma, dt))
    return u, up


def step_temperature(T, loads, Qr, Vn, rho, ctab, wb, cb, Ta, Qm, dt, td=False):
    T = f64(T).copy()
    _chk(lib().oracle_step_temperature(T.size, P(T), P(f64(loads)), P(f64(Qr)), P(f64(Vn)), rho, len(ctab),
                                       P(f64([a for a, _ in ctab])), P(f64([b for _, b in ctab])),
                                       wb, cb, Ta, Qm, dt, int(td)))
    return T
