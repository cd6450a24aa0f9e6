"""Instance construction on the device (mp_cc_instance) against the
reference-generated fixtures and the numpy restatement: d exact, w within
the device log's accuracy (a few ulp)."""

import numpy as np
import pytest

from conftest import golden
from oracle import oracle
from paper_1901_10084_b200 import graphs

pytestmark = pytest.mark.gpu

ULP_RTOL = 4.5e-16  # 2 ulp


@pytest.mark.parametrize("seed", [3, 4, 5])
def test_device_instance_matches_reference(tmp_path, seed):
    g = golden("graphs")
    p = tmp_path / "g.txt"
    p.write_text("".join(f"{u} {v}\n" for u, v in g[f"s{seed}_edges"]))
    comp = graphs.largest_component(graphs.load_edge_list(str(p)))
    inst = graphs.cc_instance(comp, epsilon=0.2)
    assert np.array_equal(inst.d_flat, g[f"s{seed}_d"])
    np.testing.assert_allclose(inst.w_flat, g[f"s{seed}_w"], rtol=ULP_RTOL, atol=0)


@pytest.mark.parametrize("n,p", [(3000, 0.004), (1500, 0.05)])
def test_device_instance_large_random_graph(n, p):
    rng = np.random.default_rng(n)
    a = np.triu(rng.random((n, n)) < p, 1)
    adj = [[] for _ in range(n)]
    for u, v in zip(*np.nonzero(a)):
        adj[u].append(int(v))
        adj[v].append(int(u))
    g = graphs.Graph(n=n, adj=[sorted(x) for x in adj])
    inst = graphs.cc_instance(g, epsilon=0.2)
    rowptr, cols = g.csr()
    d, w = oracle.cc_instance_np(rowptr, cols, n)
    assert np.array_equal(inst.d_flat, d)
    np.testing.assert_allclose(inst.w_flat, w, rtol=ULP_RTOL, atol=0)
    assert np.all(inst.w_flat > 0)
