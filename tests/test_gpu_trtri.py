"""GPU: the recursive lower-triangular inverse (trtri.cu) used by the fused
fit (L_P^-1, isdf.hpp:143) and the SMW core (Q^-1, smw.hpp:61) against
numpy — ragged sizes around the 128 leaf and the 2x2 levels, a padded leading
dimension, the untouched upper triangle and the singular-factor error."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _lower(n, seed):
    rng = np.random.default_rng(seed)
    a = np.tril(rng.standard_normal((n, n))) / np.sqrt(n)
    a[np.diag_indices(n)] = 1.0 + rng.random(n)
    return a


@pytest.mark.parametrize("n,ld", [(1, 1), (5, 5), (31, 33), (127, 127), (128, 128), (129, 130), (300, 300),
                                  (513, 520), (1024, 1024), (1100, 1100)])
def test_trtri_matches_numpy(n, ld):
    import torch

    from paper_2403_12340_b200 import lrgw

    a = _lower(n, n)
    full = np.full((ld, n), 7.0)
    full[:n, :n] = a + np.triu(np.full((n, n), 3.0), 1)  # upper junk must survive
    dev = torch.from_numpy(full.T.copy()).cuda().t()  # (ld, n) column-major
    view = dev[:n, :]
    lrgw.trtri_lower_dev(view)
    out = view.cpu().numpy()
    want = np.linalg.inv(a)
    got = np.tril(out)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12
    assert np.array_equal(np.triu(out, 1), np.triu(np.full((n, n), 3.0), 1))


def test_trtri_singular():
    import torch

    from paper_2403_12340_b200 import lrgw

    a = _lower(200, 3)
    a[150, 150] = 0.0
    dev = torch.from_numpy(a.T.copy()).cuda().t()
    with pytest.raises(lrgw.SingularMatrix):
        lrgw.trtri_lower_dev(dev)
