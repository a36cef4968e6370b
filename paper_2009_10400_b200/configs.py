"""The BASELINE.json workloads, as Problems.

cfg1  H8 10^3 unit cube, central source, 1000 steps (the reference CPU run)
cfg2  T4 Kuhn n=20 on [0,0.05]^3 (48k el), helical per-element fibres, TD
cfg3  liver-shaped T4 ~100k el, 3 RFA sources, perfusion, TD, dt = 0.2 ms
cfg4  H8 100^3 on [0,0.1]^3 (1M el), hourglass + Prony, TD + expansion
cfg5  H8 n^3 / T4 Kuhn ladder up to 16M elements (same physics as cfg4)
"""
from __future__ import annotations

import math

import numpy as np

from . import meshgen
from .problem import (COUPLED, EXP_ISOTROPIC, H8, T4, Prescribed, Problem, SourceRegion)

# Table 5: liver tissue.
T5 = dict(
    mu=1190.476, kappa=19444.444, eta_a=2 * 1190.476, fiber=(1.0, 0.0, 0.0),
    prony_phi=[0.5], prony_tau=[0.58], density=1060.0,
    c_table=[(37.0, 3600.0), (90.0, 4300.0)], k_table=[(37.0, 0.53), (90.0, 0.75)],
    perfusion_rate=26.6, blood_specific_heat=3617.0, arterial_temperature=37.0, metabolic_rate=33800.0,
    expansion=dict(kind=EXP_ISOTROPIC, alpha_i=1e-4, reference_temperature=37.0),
)
Q_R_TABLE5 = 9_705_360.0


def ramp_time(length, dt, steps):
    """Prescribed-displacement ramp: over the run, but never faster than
    ten dilatational wave transits of the block — a shorter run must not turn the
    quasi-static pull into an impact that inverts elements."""
    cd = math.sqrt((T5["kappa"] + 4 * T5["mu"] / 3) / T5["density"])
    return max(dt * steps, 10.0 * length / cd)


def _faces(nodes, axis, value, tol=1e-12):
    return np.nonzero(np.abs(nodes[:, axis] - value) <= tol)[0].astype(np.int32)


def _base(kind, nodes, el, dt, steps, **kw):
    params = dict(T5)
    params.update(kw)
    return Problem(kind=kind, nodes=nodes, elements=el, dt=dt, duration=dt * steps,
                   mode=COUPLED, expansion_enabled=True, temperature_dependent=True,
                   damping_gamma=1.0, hourglass_stiffness=0.1, **params)


def cube_problem(kind, n, length, dt, steps, top_uz, source_diameter, prony_terms=1, **kw):
    """Structured cube (H8 n^3 or T4 Kuhn n^3): bottom fixed, top u_z ramped over the run,
    central spherical source (Appendix D 'Loads')."""
    if kind == H8:
        nodes, el = meshgen.structured_h8(n, length)
    else:
        nodes, el = meshgen.kuhn_t4(n, length)
    p = _base(kind, nodes, el, dt, steps, **kw)
    if prony_terms == 2:
        p.prony_phi, p.prony_tau = [0.3, 0.2], [0.58, 0.058]
    elif prony_terms == 0:
        p.prony_phi, p.prony_tau = [], []
    p.fixed_nodes = _faces(nodes, 2, 0.0)
    p.prescribed = [Prescribed(_faces(nodes, 2, length, tol=1e-9 * length), 2, top_uz, ramp_time(length, dt, steps))]
    src = meshgen.elements_in_sphere(nodes, el, [0.5 * length] * 3, source_diameter)
    p.sources = [SourceRegion(src, Q_R_TABLE5)]
    return p


def cfg1(steps=1000):
    return cube_problem(H8, 10, 1.0, 0.01, steps, 0.1, 0.2)


def cfg2(steps=1000, n=20):
    p = cube_problem(T4, n, 0.05, 2.5e-4, steps, 5e-3, 0.01)
    zc = meshgen.centroids(p.nodes, p.elements)[:, 2]
    L = 0.05
    p.fiber_dirs = np.stack([np.cos(math.pi * zc / L), np.sin(math.pi * zc / L), np.zeros_like(zc)], axis=1)
    return p


def cfg3(steps=1000, target_elements=100_000):
    nodes, el, h = meshgen.liver_t4(target_elements)
    p = _base(T4, nodes, el, 2e-4, steps)
    xmax = nodes[:, 0].max()
    p.fixed_nodes = np.nonzero(nodes[:, 0] >= xmax - 0.01)[0].astype(np.int32)
    p.sources = [SourceRegion(meshgen.elements_in_sphere(nodes, el, c, 0.01), Q_R_TABLE5)
                 for c in ((-0.01, 0.0, 0.0), (0.0, 0.0, 0.0), (0.01, 0.0, 0.0))]
    return p


def cfg4(steps=200, n=100, prony_terms=1):
    return cube_problem(H8, n, 0.1, 1e-4, steps, 1e-2, 0.01, prony_terms=prony_terms)


def cfg4_jittered(steps=200, half=0, seed=6):
    """cfg4 with its nodes jittered by up to 5 % of the spacing, so its elements are not affine
    (the general H8 hourglass path); half=1: only the nodes in the upper half in x, a mesh of affine and
    general elements with mixed chunks along the interface."""
    p = cfg4(steps=steps)
    h = 0.1 / 100
    d = np.random.default_rng(seed).uniform(-0.05 * h, 0.05 * h, p.nodes.shape)
    if half:
        x = p.nodes[:, 0]
        d[x <= 0.5 * (x.min() + x.max()) + 1e-12] = 0.0
    p.nodes = p.nodes + d
    return p


def cfg5_h8(n, steps=50):
    """Ladder point n in {100,126,159,200,252}: dt = half the mechanical critical step."""
    length = 0.1 * n / 100
    h = length / n
    cd = math.sqrt((T5["kappa"] + 4 * T5["mu"] / 3) / T5["density"])
    dt = 0.5 * 0.9 * h / cd
    return cube_problem(H8, n, length, dt, steps, 1e-2 * n / 100, 0.01 * n / 100)


def cfg5_t4(n, steps=50):
    length = 0.1 * n / 100
    h = length / n
    cd = math.sqrt((T5["kappa"] + 4 * T5["mu"] / 3) / T5["density"])
    dt = 0.5 * 0.9 * h / cd
    return cube_problem(T4, n, length, dt, steps, 1e-2 * n / 100, 0.01 * n / 100)


def small_problem(kind=H8, n=4, steps=20, seed=0, perturb=True, **kw):
    """A tiny, strongly non-linear case for kernel parity: perturbed start and random
    per-element fibres (Appendix D 'Variants')."""
    length = 0.01 * n
    h = length / n
    cd = math.sqrt((T5["kappa"] + 4 * T5["mu"] / 3) / T5["density"])
    dt = 0.4 * 0.9 * h / cd
    p = cube_problem(kind, n, length, dt, steps, 0.1 * length, 0.5 * length, **kw)
    rng = np.random.default_rng(seed)
    if perturb:
        f = rng.normal(size=(p.num_elements, 3))
        p.fiber_dirs = f / np.linalg.norm(f, axis=1, keepdims=True)
    return p
