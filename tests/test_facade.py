"""The C++ facade (include/tve_gpu.hpp): a reference-shaped caller compiles against
the C ABI (CPU) and, on a GPU, reproduces the oracle's cfg1 summary."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2009_10400_b200", "lib")
BIN = os.path.join(ROOT, "build", "facade_demo")


def compile_demo():
    os.makedirs(os.path.dirname(BIN), exist_ok=True)
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    subprocess.run([cxx, "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "facade_demo.cpp"), "-L", LIBDIR, "-ltvegpu",
                    f"-Wl,-rpath,{LIBDIR}", "-o", BIN], check=True)


def test_facade_compiles_and_links():
    compile_demo()
    assert os.path.exists(BIN)


def test_c_header_is_plain_c():
    """tvegpu.h must compile as C (the FFI boundary carries no C++ types)."""
    src = os.path.join(ROOT, "build", "abi_check.c")
    os.makedirs(os.path.dirname(src), exist_ok=True)
    with open(src, "w") as f:
        f.write('#include "tvegpu.h"\nint main(void) { tvegpu_options o; tvegpu_default_options(&o); '
                'return tvegpu_abi_version() == TVEGPU_ABI_VERSION ? 0 : 1; }\n')
    cc = "/usr/bin/gcc" if os.path.exists("/usr/bin/gcc") else "gcc"
    out = os.path.join(ROOT, "build", "abi_check")
    subprocess.run([cc, "-std=c99", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR,
                    "-ltvegpu", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    assert subprocess.run([out]).returncode == 0


@pytest.mark.gpu
def test_facade_demo_matches_oracle():
    from oracle import oracle as O
    from paper_2009_10400_b200 import configs
    compile_demo()
    steps = 200
    out = subprocess.run([BIN, str(steps)], capture_output=True, text=True, check=True).stdout
    m = re.search(r"T_max ([0-9.eE+-]+)\s+u_z \[([0-9.eE+-]+), ([0-9.eE+-]+)\]", out)
    assert m, out
    Tmax, uzmax = float(m.group(1)), float(m.group(3))
    p = configs.cfg1(steps=steps)
    o = O.OracleEngine(p)
    o.step(steps)
    s = o.state()
    assert abs(Tmax - s["T"].max()) <= 1e-10 * (s["T"].max() - 37.0)
    assert abs(uzmax - s["u"][2::3].max()) <= 1e-10 * abs(s["u"]).max()
    assert "after reset + 1 step" in out
    assert "checkpoint resume bit-identical: yes" in out
    assert "run(): 50 steps, 5 snapshots" in out
    m = re.search(r"device summary: T_max ([0-9.eE+-]+)\s+u_z max ([0-9.eE+-]+)\s+ablation\(40C\) ([0-9.eE+-]+) m\^3 "
                  r"in (\d+) elements", out)
    assert m, out
    assert float(m.group(1)) == Tmax  # device reduction == host max of the same field
    vo, no = O.ablation_volume("H8", p.nodes, p.elements, s["T"], 40.0, disp=s["u"])
    assert int(m.group(4)) == no and abs(float(m.group(3)) - vo) <= 1e-9 * max(vo, 1e-30)


def test_facade_load_mesh_on_cpu():
    """tve::gpu::load_mesh (mesh.hpp:76) from C++: host-only, runs without a GPU."""
    src = os.path.join(ROOT, "build", "load_mesh_check.cpp")
    with open(src, "w") as f:
        f.write(r'''#include <cstdio>
#include "tve_gpu.hpp"
int main() {
    const char* text = "# unit cube\n$nodes 8\n1 0 0 0\n2 1 0 0\n3 1 1 0\n4 0 1 0\n5 0 0 1\n6 1 0 1\n7 1 1 1\n8 0 1 1\n"
                       "$elements 1 h8\n1 1 2 3 4 5 6 7 8\n$nodeset bottom 4\n1 2 3 4\n";
    tve::gpu::Mesh m = tve::gpu::load_mesh(text);
    std::printf("%d %d %d %zu\n", m.node_count(), m.element_count(), m.elements[0][6], m.node_sets["bottom"].size());
    try { tve::gpu::load_mesh("$nodes 1\n1 0 0\n"); } catch (const tve::gpu::ParseError& e) { std::printf("parse: %s\n", e.what()); }
    return 0;
}
''')
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else "g++"
    out = os.path.join(ROOT, "build", "load_mesh_check")
    subprocess.run([cxx, "-std=c++17", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), src, "-L", LIBDIR,
                    "-ltvegpu", f"-Wl,-rpath,{LIBDIR}", "-o", out], check=True)
    res = subprocess.run([out], capture_output=True, text=True, check=True).stdout.splitlines()
    assert res[0] == "8 1 6 4"
    assert res[1].startswith("parse: line 2")
