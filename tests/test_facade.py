"""The C++ facade (include/detlsh_b200.hpp) restores the reference's C++ API over
the C ABI.  CPU: it compiles and links against the in-tree library.  GPU: a
program written against it returns the oracle's exact answers."""
import os
import subprocess

import numpy as np
import pytest

from oracle.bindings import make_params

HERE = os.path.dirname(os.path.abspath(__file__))
CPP = os.path.join(HERE, "cpp")
DEMO = os.path.join(CPP, "facade_demo")


def lcg_data(n, nq, d):
    s = 12345
    out = np.empty((n + nq) * d, np.float32)
    m = (1 << 64) - 1
    for i in range(out.size):
        s = (s * 6364136223846793005 + 1442695040888963407) & m
        out[i] = (s >> 40) % 256
    out = out.reshape(n + nq, d)
    return out[:n], out[n:]


def test_facade_compiles_and_links():
    subprocess.run(["make", "-s", "-C", CPP], check=True)
    assert os.path.exists(DEMO)


@pytest.mark.gpu
def test_facade_reference_signatures_match_reference(ref):
    """build_index(shared_ptr<const Dataset>, ...), DetIndex::family/table/trees/
    project_query, estimate_rmin and the range queries through the facade."""
    if not os.path.exists(DEMO):
        subprocess.run(["make", "-s", "-C", CPP], check=True)
    out = subprocess.run([DEMO], check=True, capture_output=True, text=True).stdout.splitlines()
    f = {x.split()[0]: x.split()[1:] for x in out if x.split()[0] in ("dataset_build", "estimate_rmin", "range")}
    same, ncoef, ntab, ntrees = map(int, f["dataset_build"])
    assert same == 1 and ncoef == 4 * 16 * 24 and ntab == 4 * 16 * 257 and ntrees == 4
    base, Q = lcg_data(5000, 5, 24)
    ri = ref.build_index(base, make_params(beta=0.1, k=7, leaf_capacity=32), 77)
    assert float(f["estimate_rmin"][0]) == ri.estimate_rmin(Q[:3], 7)
    qp = ri.project_query(Q[0], 1)
    rad = ri.params.epsilon * ri.params.r_min
    drained = ri.range_query(1, qp, rad, 40)
    exact = ri.range_query(1, qp, rad, exact=True)
    assert int(f["range"][0]) == len(drained) and int(f["range"][1]) == len(exact)
    assert [int(x) for x in f["range"][2:]] == drained[:5].tolist()


@pytest.mark.gpu
def test_facade_program_matches_oracle(port):
    if not os.path.exists(DEMO):
        subprocess.run(["make", "-s", "-C", CPP], check=True)
    out = subprocess.run([DEMO], check=True, capture_output=True, text=True).stdout.splitlines()
    r_min = float(out[0].split()[1])
    detl = [x.split() for x in out if x.startswith("detl ")]
    assert detl and int(detl[0][1]) > 0 and detl[0][2] == "DETL"
    rows = [tuple(x.split()) for x in out[1:] if x.split()[0].isdigit()]
    base, Q = lcg_data(5000, 5, 24)
    oi = port.build_index(base, make_params(beta=0.1, k=7, leaf_capacity=32), 77)
    assert r_min == oi.params.r_min
    for qi in range(5):
        ids, ds, _, _ = oi.ck_ann(Q[qi], 7)
        got = [(int(r[2]), float(r[3])) for r in rows if int(r[0]) == qi]
        assert [g[0] for g in got] == ids.tolist()
        assert [g[1] for g in got] == ds.tolist()
