"""GPU unit checks of the batched dense kernels behind the hot path, against plain numpy
float64 references: the Gauss-Jordan pivot inverse (reading R16) in its three variants —
shared-memory (n <= 160), blocked single-CTA panels, blocked 8-CTA cluster panels (few large
matrices: the top system) — on saddle-point matrices [[K, U], [V^T, 0]] that need pivoting."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2301_12704_b200 import aifmm as G  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    G.load()
    yield


def _saddle(m, k, seed):
    rng = np.random.default_rng(seed)
    K = rng.standard_normal((m, m)) + 4 * np.eye(m)
    U = np.linalg.qr(rng.standard_normal((m, k)))[0]
    V = np.linalg.qr(rng.standard_normal((m, k)))[0]
    P = np.zeros((m + k, m + k))
    P[:m, :m], P[:m, m:], P[m:, :m] = K, U, V.T
    return P


@pytest.mark.parametrize("m,k", [(1, 0), (20, 13), (64, 60), (100, 61), (250, 90), (700, 300), (1100, 243)])
def test_pivot_inverse_matches_numpy(m, k):
    P = _saddle(m, k, m + k)
    Gi = G.debug_inverse(torch.from_numpy(P).cuda()).cpu().numpy()
    ref = np.linalg.inv(P)
    cond = np.linalg.cond(P)
    assert np.linalg.norm(Gi - ref) <= 1e-14 * cond * np.linalg.norm(ref) * np.sqrt(m + k)
    assert np.linalg.norm(P @ Gi - np.eye(m + k)) <= 1e-12 * cond


def test_singular_pivot_reported():
    P = _saddle(50, 10, 3)
    P[:, 7] = 0.0
    with pytest.raises(G.AIFMMError) as e:
        G.debug_inverse(torch.from_numpy(P).cuda())
    assert e.value.code == -5
