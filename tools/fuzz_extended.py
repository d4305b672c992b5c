"""Extended randomised parity sweep: the cases of tests/test_gpu_fuzz.py for
many more seeds (default + HILO field + large instances), reporting failures
instead of stopping.  Usage: python tools/fuzz_extended.py [n_cases]"""
import os
import sys
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import test_gpu_fuzz as F  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 400
fails = []
for name, fn, cases in [("default", F.test_random_instance_matches_oracle, range(96, 96 + N)),
                        ("hilo", F.test_random_instance_hilo_field, range(48, 48 + N // 2)),
                        ("large", F.test_random_large_instance_matches_oracle, range(12, 12 + N // 10)),
                        ("ground", F.test_random_ground_state_matches_oracle, range(24, 24 + N // 4))]:
    ok = 0
    for k in cases:
        try:
            fn(k)
            ok += 1
        except Exception as e:  # noqa: BLE001
            fails.append((name, k, repr(e)[:300]))
            traceback.print_exc(limit=1)
    print(f"{name}: {ok}/{len(cases)} passed", flush=True)
print("FAILURES:", len(fails))
for f in fails:
    print(f)
