"""The command-line entry point over the C++ facade:
config parsing / validation and `check` on the CPU, `run`, `verify`, `bench` on a GPU.
Exit codes: 0 success, 1 config / validation, 2 instability, 3 verification failure."""
import json
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

from paper_2009_10400_b200 import meshgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2009_10400_b200", "lib")
BIN = os.path.join(ROOT, "build", "tve_gpu")

CFG = """# Table-5 liver tissue, one spherical RF source, bottom fixed, top pressed
[mesh]
file = block.mesh
[material]
mu = 1190.476
kappa = 19444.444
fiber = 1 0 0
[thermal]
density = 1060
specific_heat = 37:3600, 90:4300
conductivity = 37:0.53, 90:0.75
perfusion_rate = 26.6
blood_specific_heat = 3617
metabolic_rate = 33800
[expansion]
kind = isotropic
alpha_i = 1e-4
[viscoelastic]
prony = 0.5:0.58
[sources]
sphere = 0.01 0.01 0.01 0.006 9705360
[bcs]
fixed = bottom
prescribed = top 2 -0.0005 0.5
[sim]
dt = 0.0002
duration = 0.02
expansion = on
temperature_dependent = on
damping_gamma = 1.0
[output]
snapshot_interval = 0.01
probe_nodes = 1 666
ablation_threshold = 40
"""


_BUILT = []


def build():
    if _BUILT:
        return
    _BUILT.append(True)
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tools", "tve_gpu_cli.cpp"), "-L", LIBDIR, "-ltvegpu",
                    f"-Wl,-rpath,{LIBDIR}", "-o", BIN], check=True)


def write_case(d, n=10, L=0.02, cfg=CFG, flip_first=False):
    nodes, el = meshgen.structured_h8(n, L)
    if flip_first:
        el = el.copy()
        el[0] = el[0][[4, 5, 6, 7, 0, 1, 2, 3]]  # upside down: inverted
    lines = [f"$nodes {len(nodes)}"] + [f"{i + 1} {float(x)!r} {float(y)!r} {float(z)!r}"
                                        for i, (x, y, z) in enumerate(nodes)]
    lines += [f"$elements {len(el)} h8"] + [f"{e + 1} " + " ".join(str(v + 1) for v in el[e]) for e in range(len(el))]
    bot, top = np.nonzero(nodes[:, 2] < 1e-9)[0], np.nonzero(nodes[:, 2] > L - 1e-9)[0]
    lines += [f"$nodeset bottom {len(bot)}", " ".join(str(i + 1) for i in bot),
              f"$nodeset top {len(top)}", " ".join(str(i + 1) for i in top)]
    (d / "block.mesh").write_text("\n".join(lines) + "\n")
    (d / "demo.cfg").write_text(cfg)
    return nodes, el


def cli(*args, cwd=None):
    return subprocess.run([BIN, *args], capture_output=True, text=True, cwd=cwd)


def test_check_reports_dofs_and_critical_steps(tmp_path):
    build()
    nodes, el = write_case(tmp_path)
    r = cli("check", "--config", str(tmp_path / "demo.cfg"), "--json")
    assert r.returncode == 0, r.stderr
    d = json.loads(r.stdout)
    assert d["dofs"] == 4 * len(nodes) and d["elements"] == len(el)
    assert abs(d["volume_m3"] - 0.02 ** 3) < 1e-18
    assert 0 < d["dt_mechanical"] < d["dt_thermal"]


@pytest.mark.parametrize("edit,err", [
    (("[sim]\n", "[sim]\nbogus = 1\n"), "unknown key 'bogus'"),
    (("dt = 0.0002\n", ""), "missing required key sim.dt"),
    (("[output]\n", "[outputs]\n"), "unknown section"),
    (("dt = 0.0002\n", "dt = 0.5\n"), "exceeds the critical step"),
])
def test_config_errors_exit_1(tmp_path, edit, err):
    build()
    write_case(tmp_path, cfg=CFG.replace(*edit))
    r = cli("check", "--config", str(tmp_path / "demo.cfg"))
    assert r.returncode == 1 and err in r.stderr, r.stderr


def test_inverted_element_exit_1_naming_it(tmp_path):
    build()
    write_case(tmp_path, flip_first=True)
    r = cli("check", "--config", str(tmp_path / "demo.cfg"))
    assert r.returncode == 1 and "element 1" in r.stderr, r.stderr


def test_override_and_verify_list(tmp_path):
    build()
    write_case(tmp_path)
    r = cli("check", "--config", str(tmp_path / "demo.cfg"), "--override", "sim.dt=1e-5", "--json")
    assert r.returncode == 0 and json.loads(r.stdout)["dt"] == 1e-5
    r = cli("verify", "--list")
    assert r.returncode == 0 and r.stdout.split() == ["perfusion_decay", "slab_conduction", "free_expansion",
                                                       "stress_relaxation"]


@pytest.mark.gpu
def test_run_writes_outputs(tmp_path):
    build()
    nodes, el = write_case(tmp_path)
    out = tmp_path / "out"
    r = cli("run", "--config", str(tmp_path / "demo.cfg"), "--out", str(out), "--json")
    assert r.returncode == 0, r.stderr
    s = json.loads(r.stdout)
    assert s["steps"] == 100 and s["max_temperature"] > 37.0 and s["min_disp"][2] < 0
    snaps = sorted(p.name for p in out.glob("snapshot_*.vtk"))
    assert snaps == ["snapshot_00000000.vtk", "snapshot_00000050.vtk", "snapshot_00000100.vtk"]
    text = (out / "snapshot_00000100.vtk").read_text().splitlines()
    i = text.index("SCALARS temperature double 1")
    T = np.array([float(v) for v in text[i + 2:i + 2 + len(nodes)]])
    assert abs(T.max() - s["max_temperature"]) <= 1e-8 * s["max_temperature"]  # 9 significant digits
    probes = (out / "probes.csv").read_text().splitlines()
    assert probes[0] == "time,node_id,T,ux,uy,uz" and len(probes) == 1 + 3 * 2
    abl = (out / "ablation.csv").read_text().splitlines()
    assert abl[0] == "time,threshold,volume_m3,elements_above" and len(abl) == 4
    r = cli("run", "--config", str(tmp_path / "demo.cfg"), "--out", str(tmp_path / "o2"), "--json",
            "--override", "sim.coupling=thermal_only")
    s2 = json.loads(r.stdout)  # displacement extrema all zero
    assert r.returncode == 0 and s2["min_disp"] == [0, 0, 0] and s2["max_disp"] == [0, 0, 0]


@pytest.mark.gpu
def test_instability_exit_2(tmp_path):  # SPEC.md:477 (explicit heat equation far above its critical step)
    build()
    cfg = CFG.replace("dt = 0.0002\n", "dt = 100\nallow_unstable_dt = on\ncoupling = thermal_only\n").replace(
        "duration = 0.02\n", "duration = 100000\n").replace("snapshot_interval = 0.01", "snapshot_interval = 0")
    write_case(tmp_path, cfg=cfg)
    r = cli("run", "--config", str(tmp_path / "demo.cfg"), "--out", str(tmp_path / "o"))
    assert r.returncode == 2 and "instability at step" in r.stderr, (r.returncode, r.stderr)


@pytest.mark.gpu
def test_verify_all_pass_and_bench():
    build()
    r = cli("verify")
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count(",yes") == 4
    r = cli("bench", "--mesh-kind", "h8", "--steps", "20")
    assert r.returncode == 0, r.stderr
    assert "scaling slope" in r.stdout and len(r.stdout.strip().splitlines()) == 7


TET_CFG = """# single tet at rest: no sources, no metabolism, blood at the initial temperature
[mesh]
file = tet.mesh
[material]
mu = 1190.476
kappa = 19444.444
[thermal]
density = 1060
specific_heat = 3600
conductivity = 0.53
perfusion_rate = 26.6
blood_specific_heat = 3617
metabolic_rate = 0
[sim]
dt = 0.0001
duration = 0.0003
[output]
snapshot_interval = 0.0001
"""


@pytest.mark.gpu
def test_single_tet_snapshot_golden(tmp_path):  # SPEC.md:432-434 write_snapshot examples
    build()
    (tmp_path / "tet.mesh").write_text("$nodes 4\n1 0 0 0\n2 0.01 0 0\n3 0 0.01 0\n4 0 0 0.01\n"
                                       "$elements 1 t4\n1 1 2 3 4\n")
    (tmp_path / "tet.cfg").write_text(TET_CFG)
    out = tmp_path / "out"
    r = cli("run", "--config", str(tmp_path / "tet.cfg"), "--out", str(out), "--json")
    assert r.returncode == 0, r.stderr
    # golden-file stable: byte-identical to the committed fixture (9 significant digits)
    golden = (Path(ROOT) / "tests" / "golden" / "single_tet_snapshot.vtk").read_bytes()
    assert (out / "snapshot_00000000.vtk").read_bytes() == golden
    # distinct files named by the zero-padded step index
    snaps = sorted(p.name for p in out.glob("snapshot_*.vtk"))
    assert snaps == [f"snapshot_{k:08d}.vtk" for k in range(4)]
    # round trip: re-parsing reproduces the arrays (the rest state stays at rest)
    text = (out / "snapshot_00000003.vtk").read_text().splitlines()
    i = text.index("SCALARS temperature double 1")
    assert [float(v) for v in text[i + 2:i + 6]] == [37.0] * 4
    j = text.index("VECTORS displacement double")
    assert [float(v) for line in text[j + 1:j + 5] for v in line.split()] == [0.0] * 12
