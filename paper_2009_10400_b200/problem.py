"""Problem description mirroring the reference's setup types, and its flat C view.

The reference builds an engine from ``Mesh`` (mesh.hpp:22-37), ``MaterialModel``
(materials.hpp:89-97), ``MechBCs`` (mechanics.hpp:37-47), ``ThermalBCs``
(bioheat.hpp:32-35), ``HeatSourceSet`` (bioheat.hpp:28-30) and
``SimulationConfig`` (engine.hpp:28-39).  :class:`Problem` holds the same fields
as numpy arrays / scalars and produces the ``tvegpu_problem`` descriptor of
``include/tvegpu.h`` (field order must match that header exactly).  Both the
product library and the test oracle consume that same descriptor.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import math
from typing import List, Optional

import numpy as np

T4, H8 = 0, 1
COUPLED, THERMAL_ONLY, MECHANICAL_ONLY = 0, 1, 2
EXP_ISOTROPIC, EXP_TRANSVERSELY_ISOTROPIC, EXP_ORTHOTROPIC = 0, 1, 2

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)


class CPrescribed(C.Structure):
    _fields_ = [("num_nodes", C.c_int32), ("nodes", _ip), ("component", C.c_int32),
                ("target", C.c_double), ("ramp_time", C.c_double)]


class CSource(C.Structure):
    _fields_ = [("num_elements", C.c_int32), ("elements", _ip), ("q_r", C.c_double),
                ("t_start", C.c_double), ("t_end", C.c_double)]


class CProblem(C.Structure):
    _fields_ = [
        ("kind", C.c_int32), ("num_nodes", C.c_int32), ("num_elements", C.c_int32),
        ("nodes", _dp), ("elements", _ip), ("fiber_dirs", _dp), ("expansion_axes", _dp),
        ("ref_specific_heat", C.c_double),
        ("mu", C.c_double), ("kappa", C.c_double), ("eta_a", C.c_double),
        ("prony_count", C.c_int32), ("prony_phi", _dp), ("prony_tau", _dp),
        ("density", C.c_double),
        ("c_table_len", C.c_int32), ("c_table_T", _dp), ("c_table_value", _dp),
        ("k_table_len", C.c_int32), ("k_table_T", _dp), ("k_table_tensor", _dp),
        ("perfusion_rate", C.c_double), ("blood_specific_heat", C.c_double),
        ("arterial_temperature", C.c_double), ("metabolic_rate", C.c_double),
        ("has_expansion", C.c_int32), ("expansion_kind", C.c_int32),
        ("alpha_i", C.c_double), ("alpha_m", C.c_double), ("alpha_n", C.c_double),
        ("reference_temperature", C.c_double),
        ("has_fiber", C.c_int32), ("fiber", C.c_double * 3), ("axis_m", C.c_double * 3),
        ("axis_n", C.c_double * 3),
        ("num_fixed_nodes", C.c_int32), ("fixed_nodes", _ip),
        ("num_prescribed", C.c_int32), ("prescribed", C.POINTER(CPrescribed)),
        ("external_force", _dp), ("body_force", C.c_double * 3),
        ("num_fixed_temperatures", C.c_int32), ("fixed_temperature_nodes", _ip),
        ("fixed_temperature_values", _dp), ("initial_temperature", C.c_double),
        ("num_sources", C.c_int32), ("sources", C.POINTER(CSource)),
        ("dt", C.c_double), ("duration", C.c_double), ("mode", C.c_int32),
        ("expansion_enabled", C.c_int32), ("temperature_dependent", C.c_int32),
        ("damping_gamma", C.c_double), ("hourglass_stiffness", C.c_double),
        ("allow_unstable_dt", C.c_int32), ("workers", C.c_int32),
    ]


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


@dataclasses.dataclass
class Prescribed:
    """PrescribedDisplacement (mechanics.hpp:25-35)."""
    nodes: np.ndarray
    component: int
    target: float
    ramp_time: float = 0.0

    def value_at(self, t: float) -> float:
        if self.ramp_time <= 0:
            return self.target
        return self.target * min(t / self.ramp_time, 1.0)


@dataclasses.dataclass
class SourceRegion:
    """SourceRegion (bioheat.hpp:19-26)."""
    elements: np.ndarray
    q_r: float
    t_start: float = 0.0
    t_end: float = math.inf


@dataclasses.dataclass
class Problem:
    # Mesh (mesh.hpp:22-37)
    kind: int
    nodes: np.ndarray                     # (N, 3)
    elements: np.ndarray                  # (E, nn)
    fiber_dirs: Optional[np.ndarray] = None       # (E, 3)
    expansion_axes: Optional[np.ndarray] = None   # (E, 6)
    # HyperelasticParams / PronySeries (materials.hpp:15-36)
    mu: float = 1190.476
    kappa: float = 19444.444
    eta_a: float = 0.0
    prony_phi: List[float] = dataclasses.field(default_factory=list)
    prony_tau: List[float] = dataclasses.field(default_factory=list)
    # ThermalProps (materials.hpp:67-75)
    density: float = 1060.0
    c_table: List[tuple] = dataclasses.field(default_factory=lambda: [(37.0, 3600.0)])
    k_table: List[tuple] = dataclasses.field(default_factory=lambda: [(37.0, 0.53)])  # (T, k) or (T, 3x3)
    perfusion_rate: float = 0.0
    blood_specific_heat: float = 0.0
    arterial_temperature: float = 37.0
    metabolic_rate: float = 0.0
    # ExpansionSpec (materials.hpp:80-86)
    expansion: Optional[dict] = None      # {"kind", "alpha_i", "alpha_m", "alpha_n", "reference_temperature"}
    fiber: Optional[tuple] = None
    axis_m: tuple = (1.0, 0.0, 0.0)
    axis_n: tuple = (0.0, 1.0, 0.0)
    ref_specific_heat: Optional[float] = None     # precompute(mesh, rho, c_ref); default c(37)
    # MechBCs (mechanics.hpp:37-47)
    fixed_nodes: np.ndarray = dataclasses.field(default_factory=lambda: np.zeros(0, np.int32))
    prescribed: List[Prescribed] = dataclasses.field(default_factory=list)
    external_force: Optional[np.ndarray] = None   # (N, 3)
    body_force: tuple = (0.0, 0.0, 0.0)
    # ThermalBCs (bioheat.hpp:32-35)
    fixed_temperatures: List[tuple] = dataclasses.field(default_factory=list)  # (node, T)
    initial_temperature: float = 37.0
    # HeatSourceSet (bioheat.hpp:28-30)
    sources: List[SourceRegion] = dataclasses.field(default_factory=list)
    # SimulationConfig (engine.hpp:28-39)
    dt: float = 1e-4
    duration: float = 0.0
    mode: int = COUPLED
    expansion_enabled: bool = False
    temperature_dependent: bool = False
    damping_gamma: float = 0.0
    hourglass_stiffness: float = 0.1
    allow_unstable_dt: bool = False
    workers: int = 0

    @property
    def nn(self) -> int:
        return 4 if self.kind == T4 else 8

    @property
    def num_nodes(self) -> int:
        return int(self.nodes.shape[0])

    @property
    def num_elements(self) -> int:
        return int(self.elements.shape[0])

    @property
    def prony_count(self) -> int:
        return len(self.prony_phi)

    def to_c(self):
        """Return (CProblem, keepalive) — keep ``keepalive`` referenced while the struct is used."""
        keep = []

        def hold(a):
            keep.append(a)
            return a

        p = CProblem()
        p.kind = self.kind
        p.num_nodes = self.num_nodes
        p.num_elements = self.num_elements
        p.nodes = _ptr(hold(_f64(self.nodes).reshape(-1)), _dp)
        p.elements = _ptr(hold(_i32(self.elements).reshape(-1)), _ip)
        p.fiber_dirs = _ptr(hold(_f64(self.fiber_dirs).reshape(-1)), _dp) if self.fiber_dirs is not None else None
        p.expansion_axes = (_ptr(hold(_f64(self.expansion_axes).reshape(-1)), _dp)
                            if self.expansion_axes is not None else None)
        c_tab = sorted(self.c_table)
        p.ref_specific_heat = float(self.ref_specific_heat if self.ref_specific_heat is not None
                                    else _interp(c_tab, 37.0))
        p.mu, p.kappa, p.eta_a = self.mu, self.kappa, self.eta_a
        p.prony_count = self.prony_count
        p.prony_phi = _ptr(hold(_f64(self.prony_phi)), _dp) if self.prony_count else None
        p.prony_tau = _ptr(hold(_f64(self.prony_tau)), _dp) if self.prony_count else None
        p.density = self.density
        p.c_table_len = len(c_tab)
        p.c_table_T = _ptr(hold(_f64([t for t, _ in c_tab])), _dp)
        p.c_table_value = _ptr(hold(_f64([v for _, v in c_tab])), _dp)
        k_tab = sorted(self.k_table, key=lambda e: e[0])
        p.k_table_len = len(k_tab)
        p.k_table_T = _ptr(hold(_f64([t for t, _ in k_tab])), _dp)
        tens = [np.asarray(v, np.float64) * np.eye(3) if np.ndim(v) == 0 else np.asarray(v, np.float64)
                for _, v in k_tab]
        p.k_table_tensor = _ptr(hold(_f64(np.stack(tens)).reshape(-1)), _dp)
        p.perfusion_rate = self.perfusion_rate
        p.blood_specific_heat = self.blood_specific_heat
        p.arterial_temperature = self.arterial_temperature
        p.metabolic_rate = self.metabolic_rate
        if self.expansion is not None:
            p.has_expansion = 1
            p.expansion_kind = int(self.expansion.get("kind", EXP_ISOTROPIC))
            p.alpha_i = float(self.expansion.get("alpha_i", 0.0))
            p.alpha_m = float(self.expansion.get("alpha_m", 0.0))
            p.alpha_n = float(self.expansion.get("alpha_n", 0.0))
            p.reference_temperature = float(self.expansion.get("reference_temperature", 37.0))
        if self.fiber is not None:
            p.has_fiber = 1
            p.fiber[:] = list(self.fiber)
        p.axis_m[:] = list(self.axis_m)
        p.axis_n[:] = list(self.axis_n)
        fixed = hold(_i32(self.fixed_nodes))
        p.num_fixed_nodes = fixed.size
        p.fixed_nodes = _ptr(fixed, _ip) if fixed.size else None
        if self.prescribed:
            arr = (CPrescribed * len(self.prescribed))()
            for k, q in enumerate(self.prescribed):
                nodes = hold(_i32(q.nodes))
                arr[k].num_nodes = nodes.size
                arr[k].nodes = _ptr(nodes, _ip)
                arr[k].component = q.component
                arr[k].target = q.target
                arr[k].ramp_time = q.ramp_time
            hold(arr)
            p.num_prescribed = len(self.prescribed)
            p.prescribed = C.cast(arr, C.POINTER(CPrescribed))
        p.external_force = (_ptr(hold(_f64(self.external_force).reshape(-1)), _dp)
                            if self.external_force is not None else None)
        p.body_force[:] = list(self.body_force)
        if self.fixed_temperatures:
            nodes = hold(_i32([n for n, _ in self.fixed_temperatures]))
            vals = hold(_f64([v for _, v in self.fixed_temperatures]))
            p.num_fixed_temperatures = nodes.size
            p.fixed_temperature_nodes = _ptr(nodes, _ip)
            p.fixed_temperature_values = _ptr(vals, _dp)
        p.initial_temperature = self.initial_temperature
        if self.sources:
            arr = (CSource * len(self.sources))()
            for k, s in enumerate(self.sources):
                els = hold(_i32(s.elements))
                arr[k].num_elements = els.size
                arr[k].elements = _ptr(els, _ip)
                arr[k].q_r, arr[k].t_start, arr[k].t_end = s.q_r, s.t_start, s.t_end
            hold(arr)
            p.num_sources = len(self.sources)
            p.sources = C.cast(arr, C.POINTER(CSource))
        p.dt, p.duration, p.mode = self.dt, self.duration, self.mode
        p.expansion_enabled = int(self.expansion_enabled)
        p.temperature_dependent = int(self.temperature_dependent)
        p.damping_gamma = self.damping_gamma
        p.hourglass_stiffness = self.hourglass_stiffness
        p.allow_unstable_dt = int(self.allow_unstable_dt)
        p.workers = self.workers
        return p, keep


def _interp(tab, T):
    if len(tab) == 1 or T <= tab[0][0]:
        return tab[0][1]
    if T >= tab[-1][0]:
        return tab[-1][1]
    for (t0, v0), (t1, v1) in zip(tab[:-1], tab[1:]):
        if t0 <= T < t1:
            return v0 + (v1 - v0) * ((T - t0) / (t1 - t0))
    return tab[-1][1]
