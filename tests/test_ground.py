"""Exact enumerator (brute_force_ground, metrics.py:53-67) against the
reference's own outputs (tests/golden/ground.npz, make_golden_ground.py)."""

import numpy as np
import pytest

import nmfa_oracle as O

NAMES = ["pair", "single_h", "triangle", "moebius16", "cubic24_s5", "sk20_s3", "sk26_s1",
         "dense18_p05", "sk22_inth", "w2_18", "real16_h"]


@pytest.fixture(scope="module")
def G():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "ground.npz"))


def oprob(G, name):
    return O.problem_from_edges(int(G[name + "_n"]), G[name + "_ei"], G[name + "_ej"],
                                G[name + "_w"], G[name + "_h"])


@pytest.mark.parametrize("name", [n for n in NAMES if n not in ("sk26_s1", "cubic24_s5", "sk22_inth")])
def test_oracle_matches_reference(G, name):
    e, c = O.gray_ground(oprob(G, name))
    assert abs(e - float(G[name + "_E"])) <= 1e-9 and c == int(G[name + "_deg"])


def test_max_exact_n_message(G):
    from paper_1806_08422_b200 import MAX_EXACT_N
    assert MAX_EXACT_N == 26
    assert str(G["too_big_msg"]) == f"exhaustive enumeration is limited to n <= 26, got n = 27"


torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_gpu_enumerator_matches_reference(G, name):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1806_08422_b200 as nb
    p = nb.IsingProblem.from_arrays(int(G[name + "_n"]), G[name + "_ei"], G[name + "_ej"],
                                    G[name + "_w"], G[name + "_h"])
    gt, cfg = nb.brute_force_ground(p, return_config=True)
    want_e, want_c = float(G[name + "_E"]), int(G[name + "_deg"])
    if np.all(G[name + "_w"] == np.round(G[name + "_w"])) and np.all(G[name + "_h"] == np.round(G[name + "_h"])):
        assert gt.energy == want_e      # integer instances: bit-exact
    else:
        assert abs(gt.energy - want_e) <= 1e-9
    assert gt.degeneracy == want_c and gt.source == "EXACT"
    # the returned configuration attains the minimum (exact energy of the oracle)
    assert abs(O.energy(oprob(G, name), cfg) - want_e) <= 1e-9


@pytest.mark.gpu
def test_gpu_enumerator_limits():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    import paper_1806_08422_b200 as nb
    with pytest.raises(ValueError, match="limited to n <= 26, got n = 27"):
        nb.brute_force_ground(nb.gen_sk(27, 0))
    gt = nb.brute_force_ground(nb.gen_sk(28, 0), max_n=28)   # beyond the reference's limit
    assert gt.degeneracy >= 2 and gt.degeneracy % 2 == 0      # global-flip pairs (h = 0)
