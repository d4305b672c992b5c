"""Native instance parser (nmfa_gset_parse) against the reference's
parse_gset outcomes (tests/golden/gset_cases.json, make_golden_gset.py):
same edges for valid texts, same message and line number for malformed ones."""

import json
import os

import numpy as np
import pytest

import paper_1806_08422_b200 as nb

CASES = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "gset_cases.json")))


@pytest.mark.parametrize("name", sorted(CASES))
def test_parse_matches_reference(name):
    c = CASES[name]
    if c["ok"]:
        p = nb.parse_gset(c["text"])
        assert p.n == c["n"]
        assert p.edges_i.tolist() == c["ei"] and p.edges_j.tolist() == c["ej"]
        assert [repr(float(x)) for x in p.edge_weights] == c["w"]
        assert np.all(p.h == 0.0)
    else:
        with pytest.raises(ValueError) as exc:
            nb.parse_gset(c["text"])
        assert str(exc.value) == c["msg"]
        if c["line"] is not None:
            assert isinstance(exc.value, nb.GsetParseError) and exc.value.line_no == c["line"]


def test_write_parse_round_trip(tmp_path):
    p = nb.gen_dense_maxcut(60, 0.3, 3)
    text = nb.write_gset(p)
    q = nb.parse_gset(text)
    assert np.array_equal(q.edges_i, p.edges_i) and np.array_equal(q.edges_j, p.edges_j)
    assert np.array_equal(q.edge_weights, p.edge_weights)
    f = tmp_path / "g.txt"
    f.write_bytes(text.encode())
    r = nb.load_gset(str(f))
    assert np.array_equal(r.edges_i, p.edges_i)
    with pytest.raises(ValueError, match="h must be zero"):
        nb.write_gset(nb.IsingProblem(2, [(0, 1, 1.0)], h=[1.0, 0.0]))


def test_load_undecodable_bytes(tmp_path):
    f = tmp_path / "bad.txt"
    f.write_bytes(b"3 1\n1 2 \xff\n")
    with pytest.raises(nb.GsetParseError) as exc:
        nb.load_gset(str(f))
    assert exc.value.line_no == 2 and "non-numeric token" in str(exc.value)


def test_large_instance_parses_fast():
    """K2000-size text (1,999,000 edge lines): the reference needs ~6.5 s."""
    import time
    p = nb.gen_sk(2000, 7)
    text = nb.write_gset(p)
    t = time.perf_counter()
    q = nb.parse_gset(text)
    dt = time.perf_counter() - t
    assert q.num_edges == p.num_edges and np.array_equal(q.edge_weights, p.edge_weights)
    assert dt < 3.0, dt


@pytest.mark.parametrize("n", [4294967296, 3037000500, (1 << 30) + 1])
def test_absurd_vertex_count_is_rejected_not_overflowed(n):
    """A header whose n * n wraps 64 bits must not size the duplicate bitset
    from the wrapped product (n = 2^32 used to segfault)."""
    with pytest.raises(nb.GsetParseError) as exc:
        nb.parse_gset(f"{n} 2\n1 2 1\n2 3 1\n")
    assert exc.value.line_no == 1 and "vertex count too large" in str(exc.value)


def test_large_n_without_bitset_still_finds_duplicates():
    """n above the bitset limit (23170) takes the sort path for duplicates."""
    with pytest.raises(nb.GsetParseError) as exc:
        nb.parse_gset("100000 3\n1 2 1\n5 9 1\n2 1 1\n")
    assert exc.value.line_no == 4 and "duplicate edge (1, 2)" in str(exc.value)
    p = nb.parse_gset("100000 2\n1 2 1\n99999 100000 -1\n")
    assert p.n == 100000 and p.edges_j.tolist() == [1, 99999]


def test_write_results_csv_matches_reference_format():
    """gset.py:107-130: header, instance id on every row, repr floats, cut from
    zero-field problems, wall_clock_us only with timings (else 0)."""
    import numpy as np

    import paper_1806_08422_b200 as nb
    p = nb.moebius_ladder(8)
    c = np.array([1.0, -1.0] * 4)
    runs = [nb.RunResult(final_config=c, final_energy=-4.0, seed=7, wall_clock=1.5e-3),
            nb.RunResult(final_config=-c, final_energy=-4.0, seed=8, wall_clock=2.5e-6)]
    w_total = float(np.sum(p.edge_weights))
    cut = repr((w_total + 4.0) * 0.5)
    got = nb.write_results_csv(runs, {"instance_id": "m8", "problem": p, "timings": True})
    assert got == ("instance_id,seed,final_energy,cut_value,wall_clock_us\n"
                   f"m8,7,-4.0,{cut},1500\nm8,8,-4.0,{cut},2\n")
    got = nb.write_results_csv(runs, {"instance_id": "m8"})
    assert got.splitlines()[1:] == ["m8,7,-4.0,,0", "m8,8,-4.0,,0"]
    hp = nb.IsingProblem(8, [(0, 1, 1.0)], h=[1.0] + [0.0] * 7)
    assert nb.write_results_csv(runs, {"problem": hp}).splitlines()[1] == ",7,-4.0,,0"
    assert nb.generators.gen_sk is nb.gen_sk and hasattr(nb.kernels, "install")
