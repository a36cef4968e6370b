"""load_mesh (mesh.hpp:73-79, SPEC.md:47-56 and the file format at SPEC.md:88): the
library's parallel parser against the SPEC examples, the stated errors, and an
independent numpy writer/reader round trip (bit-exact: both sides round correctly)."""
import numpy as np
import pytest

import paper_2009_10400_b200 as tg
from paper_2009_10400_b200 import meshgen
from paper_2009_10400_b200.problem import H8, T4


def write_mesh(nodes, el, kind, fibers=None, axes=None, node_sets=None, elem_sets=None, shuffle=None):
    rng = np.random.default_rng(shuffle) if shuffle is not None else None
    lines = ["# generated", f"$nodes {len(nodes)}"]
    order = rng.permutation(len(nodes)) if rng is not None else range(len(nodes))
    lines += [f"{i + 1} {float(nodes[i, 0])!r} {float(nodes[i, 1])!r} {float(nodes[i, 2])!r}" for i in order]
    lines.append(f"$elements {len(el)} {kind}")
    lines += [f"{e + 1} " + " ".join(str(v + 1) for v in el[e]) for e in range(len(el))]
    for name, ids in (node_sets or {}).items():
        lines.append(f"$nodeset {name} {len(ids)}")
        lines.append(" ".join(str(i + 1) for i in ids))
    for name, ids in (elem_sets or {}).items():
        lines.append(f"$elemset {name} {len(ids)}")
        lines += [str(i + 1) for i in ids]
    if fibers is not None:
        lines.append(f"$fibers {len(el)}")
        lines += [f"{e + 1} " + " ".join(repr(float(x)) for x in fibers[e]) for e in range(len(el))]
    if axes is not None:
        lines.append(f"$expansion_axes {len(el)}")
        lines += [f"{e + 1} " + " ".join(repr(float(x)) for x in axes[e]) for e in range(len(el))]
    return "\n".join(lines) + "\n"


def test_spec_unit_tet():
    m = tg.load_mesh("$nodes 4\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n$elements 1 t4\n1 1 2 3 4\n")
    assert m["kind"] == T4 and m["elements"].tolist() == [[0, 1, 2, 3]]
    assert abs(np.linalg.det((m["nodes"][1:] - m["nodes"][0]).T) / 6 - 1 / 6) < 1e-15


def test_spec_unit_cube():
    nodes, el = meshgen.structured_h8(1, 1.0)
    m = tg.load_mesh(write_mesh(nodes, el, "h8"))
    assert m["kind"] == H8
    np.testing.assert_array_equal(m["nodes"], nodes)
    np.testing.assert_array_equal(m["elements"], el)


def test_spec_out_of_range_names_element():
    with pytest.raises(tg.ValidationError, match="element 1"):
        tg.load_mesh("$nodes 4\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n$elements 1 t4\n1 1 2 3 9\n")


@pytest.mark.parametrize("text,cls,match", [
    ("$nodes 2\n1 0 0 0\n2 1 0\n$elements 1 t4\n1 1 2 1 2\n", tg.ParseError, "line 3"),
    ("$nodes 1\n1 0 0 0\n$elements 1 q9\n1 1\n", tg.ParseError, "line 3"),
    ("$nodes 4\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n$elements 1 h8\n1 1 2 3 4\n", tg.ValidationError, "mixed"),
    ("$nodes 4\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n$elements 1 t4\n1 1 3 2 4\n", tg.ValidationError,
     "inverted or degenerate element 1"),
    ("$nodes 4\n1 0 0 0\n1 1 0 0\n3 0 1 0\n4 0 0 1\n$elements 1 t4\n1 1 2 3 4\n", tg.ParseError, "duplicate"),
    ("$nodes 4\n1 0 0 0\n2 1 0 0\n3 0 1 0\n4 0 0 1\n$elements 1 t4\n1 1 2 3 4\n$fibers 1\n1 1 1 0\n",
     tg.ValidationError, "non-unit"),
    ("$bogus 3\n", tg.ParseError, "unknown section"),
])
def test_errors(text, cls, match):
    with pytest.raises(cls, match=match):
        tg.load_mesh(text)


@pytest.mark.parametrize("kind", ["t4", "h8"])
def test_round_trip_with_sets_and_directions(kind):
    nodes, el = meshgen.kuhn_t4(4, 0.04) if kind == "t4" else meshgen.structured_h8(4, 0.04)
    rng = np.random.default_rng(1)
    nodes = nodes + rng.uniform(-1e-4, 1e-4, nodes.shape)  # non-round coordinates
    f = rng.normal(size=(len(el), 3))
    f /= np.linalg.norm(f, axis=1, keepdims=True)
    a = np.concatenate([f, np.cross(f, [0.0, 0.0, 1.0])], axis=1)
    a[:, 3:] /= np.linalg.norm(a[:, 3:], axis=1, keepdims=True)
    ns = {"bottom": np.nonzero(nodes[:, 2] < 1e-3)[0], "top": np.nonzero(nodes[:, 2] > 0.039)[0]}
    es = {"src": np.arange(0, len(el), 7)}
    m = tg.load_mesh(write_mesh(nodes, el, kind, fibers=f, axes=a, node_sets=ns, elem_sets=es, shuffle=3))
    np.testing.assert_array_equal(m["nodes"], nodes)
    np.testing.assert_array_equal(m["elements"], el)
    np.testing.assert_array_equal(m["fiber_dirs"], f)
    np.testing.assert_array_equal(m["expansion_axes"], a)
    assert set(m["node_sets"]) == {"bottom", "top"} and set(m["element_sets"]) == {"src"}
    np.testing.assert_array_equal(m["node_sets"]["top"], ns["top"])
    np.testing.assert_array_equal(m["element_sets"]["src"], es["src"])


def test_file_path_and_scale(tmp_path):
    nodes, el = meshgen.structured_h8(60, 0.06)  # 216k elements
    path = tmp_path / "cube.mesh"
    path.write_text(write_mesh(nodes, el, "h8"))
    m = tg.load_mesh(str(path))
    np.testing.assert_array_equal(m["elements"], el)
    np.testing.assert_array_equal(m["nodes"], nodes)
