"""bench.py's TTS99 SK100 measurement alone (A/B of small-kernel variants via env)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_1806_08422_b200 as nb  # noqa: E402

dev = torch.device("cuda:0")
for rep in range(3):
    r = bench.measure_tts_sk100(nb, dev, skip_cpu=True)
    print(f"table={os.environ.get('NMFA_SMALL_TABLE', 'auto')} tau {r['gpu']['tau_s'] * 1e9:.1f} ns  "
          f"TTS99 {r['gpu']['tts99_s'] * 1e6:.3f} us  p {r['gpu']['p']:.4f}", flush=True)
