"""Golden parse outcomes of the REFERENCE's parse_gset (gset.py:35-89) for
valid and malformed texts.  Build container only.

    python tests/golden/make_golden_gset.py
"""
import json
import os
import sys

sys.path.insert(0, "/root/reference/pkg/src")
import nmfa  # noqa: E402
from nmfa.gset import GsetParseError, parse_gset  # noqa: E402

CASES = {
    "basic": "3 2\n1 2 1\n2 3 -1\n",
    "comments_blank": "# header next\n\n4 3\nc comment\n1 2 1\n\n# x\n2 3 2\n3 4 -3\n",
    "crlf": "3 2\r\n1 2 1\r\n3 2 5\r\n",
    "cr_only": "3 2\r1 2 1\r2 3 1\r",
    "tabs_spaces": "  3\t2  \n\t1 2   1\n 2\t3 1 \n",
    "swapped_order": "4 3\n4 1 1\n3 2 -1\n2 1 1\n",
    "numeric_forms": "4 4\n+1 2 1e0\n1_0 3 1.5\n2 3 -2.25\n1 4 1_0.5\n",
    "real_weights": "3 3\n1 2 0.5\n1 3 -1e-3\n2 3 3.25e2\n",
    "zero_edges": "5 0\n",
    "vt_ff_breaks": "3 2\x0b1 2 1\x0c2 3 1\n",
    "unicode_space": "3 2\n1 2 1\n2 3　1\n",
    "unicode_linesep": "3 2 1 2 1 2 3 1\n",
    "inf_weight_like": "3 1\n1 2 infinity\n",
    "nan_weight": "3 1\n1 2 nan\n",
    "err_empty": "",
    "err_only_comments": "# nothing\nc also nothing\n",
    "err_header_tokens": "3 2 1\n1 2 1\n",
    "err_header_nonnum": "3 x\n",
    "err_header_float": "3.0 2\n",
    "err_n_zero": "0 0\n",
    "err_m_negative": "3 -1\n",
    "err_edge_tokens": "3 1\n1 2\n",
    "err_edge_nonnum": "3 1\n1 b 1\n",
    "err_weight_nonnum": "3 1\n1 2 w\n",
    "err_range_hi": "3 1\n1 4 1\n",
    "err_range_lo": "3 1\n0 2 1\n",
    "err_huge_int": "3 1\n1 99999999999999999999999 1\n",
    "err_self_loop": "3 1\n2 2 1\n",
    "err_zero_weight": "3 1\n1 2 0.0\n",
    "err_inf_weight": "3 1\n1 2 -inf\n",
    "err_duplicate": "3 2\n1 2 1\n2 1 4\n",
    "err_duplicate_late": "4 4\n1 2 1\n3 4 1\n1 3 1\n4 3 2\n",
    "err_dup_before_count": "3 1\n1 2 1\n2 1 1\n",
    "err_more_lines": "3 1\n1 2 1\n2 3 1\n",
    "err_fewer_lines": "4 3\n1 2 1\n2 3 1\n",
    "err_first_of_two": "4 3\n1 2 1\n1 2 1\n3 3 1\n",
    "err_parse_before_dup": "4 4\n1 2 1\n2 x 1\n1 2 1\n3 4 1\n",
    "err_quote_token": "3 1\n1 2 'a'\n",
}


def main():
    out = {}
    for name, text in CASES.items():
        try:
            p = parse_gset(text)
            out[name] = {"text": text, "ok": True, "n": p.n, "ei": p.edges_i.tolist(),
                         "ej": p.edges_j.tolist(), "w": [repr(float(x)) for x in p.edge_weights]}
        except GsetParseError as e:
            out[name] = {"text": text, "ok": False, "msg": str(e), "line": e.line_no}
        except ValueError as e:  # IsingProblem validation
            out[name] = {"text": text, "ok": False, "msg": str(e), "line": None}
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "gset_cases.json"), "w") as f:
        json.dump(out, f, indent=1, ensure_ascii=True)
    print(f"wrote {len(out)} cases")


if __name__ == "__main__":
    main()
