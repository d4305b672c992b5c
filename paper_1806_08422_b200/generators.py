"""The reference's module name for the instance generators (nmfa.generators):
`from paper_1806_08422_b200.generators import gen_sk` works like
`from nmfa.generators import gen_sk`.  The implementations are in instances.py."""

from .problem import IsingProblem  # noqa: F401  (the reference module's namespace)
from .instances import (GEN_STREAM_TAG, MASK64, gen_cubic_maxcut, gen_dense_maxcut,  # noqa: F401
                        gen_sk, is_connected, moebius_ladder, toroidal_grid)
