"""Instance construction host logic (reference instance.py / tests/test_instance.py):
edge-list parsing, largest component, the numpy restatement of the Jaccard
instance against the reference-generated fixtures, and the text format."""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle
from paper_1901_10084_b200 import graphs
from paper_1901_10084_b200.graphs import Graph


def _write_edges(tmp_path, edges, name="g.txt"):
    p = tmp_path / name
    p.write_text("# seeded random graph\n" + "".join(f"{u} {v}\n" for u, v in edges))
    return str(p)


@pytest.mark.parametrize("seed", [3, 4, 5])
def test_pipeline_matches_reference_fixtures(tmp_path, seed):
    g = golden("graphs")
    path = _write_edges(tmp_path, g[f"s{seed}_edges"])
    gr = graphs.load_edge_list(path)
    comp = graphs.largest_component(gr)
    n_all, n_comp, dups, loops = g[f"s{seed}_n"].tolist()
    assert (gr.n, comp.n, gr.dropped_duplicates, gr.dropped_self_loops) == (n_all, n_comp, dups, loops)
    assert comp.labels == g[f"s{seed}_labels"].tolist()
    assert all(comp.adj[u] == sorted(comp.adj[u]) for u in range(comp.n))
    rowptr, cols = comp.csr()
    d, w = oracle.cc_instance_np(rowptr, cols, comp.n)
    assert np.array_equal(d, g[f"s{seed}_d"]) and np.array_equal(w, g[f"s{seed}_w"])


def test_jaccard_closed_neighborhoods_small():
    """reference tests/test_instance.py:45-55 through the restatement"""
    g = Graph(n=4, adj=[[1, 2], [0, 2], [0, 1, 3], [2]])
    rowptr, cols = g.csr()
    d, w = oracle.cc_instance_np(rowptr, cols, 4, offset=0.01)
    J = {(0, 1): 1.0, (0, 2): 0.75, (0, 3): 0.25, (2, 3): 0.5}
    iu = list(zip(*np.triu_indices(4, 1)))
    for (i, j), jac in J.items():
        s = np.log((1 + jac - 0.05) / (1 - jac + 0.05))
        s = np.clip(s, -10, 10)
        s = s + 0.01 if s >= 0 else s - 0.01
        p = iu.index((i, j))
        assert w[p] == pytest.approx(abs(s)) and d[p] == (1.0 if s < 0 else 0.0)


def test_edge_list_errors(tmp_path):
    p = tmp_path / "bad.txt"
    p.write_text("1 2\nnope\n")
    with pytest.raises(ValueError, match=":2:"):
        graphs.load_edge_list(str(p))
    p.write_text("1 2\n3 x\n")
    with pytest.raises(ValueError, match="non-integer"):
        graphs.load_edge_list(str(p))
    with pytest.raises(OSError):
        graphs.load_edge_list(str(tmp_path / "missing.txt"))
    with pytest.raises(ValueError):
        graphs.largest_component(Graph(n=0, adj=[]))


def test_cc_instance_argument_errors():
    g = Graph(n=6, adj=[[1], [0, 2], [1, 3], [2, 4], [3, 5], [4]])
    with pytest.raises(ValueError):
        graphs.cc_instance(g, offset=0.0)
    with pytest.raises(ValueError):
        graphs.cc_instance(Graph(n=2, adj=[[1], [0]]))


def test_instance_file_roundtrip(tmp_path):
    from paper_1901_10084_b200 import instances
    inst = instances.random_instance(7, seed=2)
    path = str(tmp_path / "inst.txt")
    graphs.save_instance(inst, path)
    assert open(path).readline().split()[:3] == ["metricinst", "1", "7"]
    back = graphs.load_instance(path)
    assert back.n == 7 and back.epsilon == inst.epsilon
    assert np.array_equal(back.d_flat, inst.d_flat) and np.array_equal(back.w_flat, inst.w_flat)
    p = tmp_path / "bad.txt"
    p.write_text("wrong 1 4 0.2\n")
    with pytest.raises(ValueError, match="bad header"):
        graphs.load_instance(str(p))
    p.write_text("metricinst 1 4 0.2\n1 2 0.0 1.0\n")
    with pytest.raises(ValueError, match="pair rows"):
        graphs.load_instance(str(p))
