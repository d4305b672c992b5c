"""The seeded in-kernel noise against its spec (oracle.device_normals).

With no couplers, h = 0, alpha = 1 and T = 1, one step gives s = -tanh(z),
so the noise each path drew is z = -atanh(s). This pins the key / counter
mapping (global replica, spin group, step), the word -> spin layout and the
Box-Muller transform on every kernel path; the statistics tests then only
have to cover the dynamics."""

import os

import numpy as np
import pytest

import nmfa_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1806_08422_b200 as nb  # noqa: E402
from paper_1806_08422_b200 import _native  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1806_08422_b200 import build
    build.build()
    _native.load()


@pytest.mark.parametrize("path,n,csr", [("small", 45, False), ("dense", 300, False),
                                        ("sparse", 300, False), ("sparse", 300, True)])
def test_seeded_noise_matches_spec(path, n, csr):
    p = nb.IsingProblem(n, [])
    p.device_handle().set_path(path)
    sigma, t_f, R, r0, seed = 0.15, 3, 70, 1000, 12345
    params = nb.NmfaParams(alpha=1.0, sigma=sigma, t_f=t_f, seed=seed)
    old = os.environ.get("NMFA_SPARSE_CSR")
    os.environ["NMFA_SPARSE_CSR"] = "1" if csr else "0"
    try:
        res = nb.sample(p, params, R, r0=r0, temps=np.ones(t_f), record_trajectory=True)
    finally:
        if old is None:
            os.environ.pop("NMFA_SPARSE_CSR", None)
        else:
            os.environ["NMFA_SPARSE_CSR"] = old
    s = res.s_hist.cpu().numpy().astype(np.float64)  # (R, t_f, n)
    z_dev = -np.arctanh(s)
    for t in range(t_f):
        z_ref = O.device_normals(seed, np.arange(r0, r0 + R), t, n, sigma)
        np.testing.assert_allclose(z_dev[:, t, :], z_ref, atol=2e-5, rtol=0)
    z = z_dev.ravel() / sigma
    assert abs(z.mean()) < 0.05 and abs(z.std() - 1.0) < 0.05
    assert np.abs(z).max() <= 5.41  # the 20-bit radius tail bound
