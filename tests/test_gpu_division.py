"""The library's call-free fp64 division (fa_div.cuh) is bitwise CUDA's __ddiv_rn."""

import numpy as np
import pytest

from paper_1305_3122_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_division_matches_ddiv_rn(seed):
    import torch

    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    first = torch.zeros(4, dtype=torch.float64, device="cuda")
    rc = _lib.lib().fa_selftest_division(20_000_000, seed, bad.data_ptr(), first.data_ptr(), _lib.stream_handle())
    _lib.check(rc)
    n_bad = int(bad.item())
    assert n_bad == 0, f"{n_bad} mismatches, e.g. x, y, mine, ref = {first.cpu().numpy().tolist()}"


def test_division_special_values_match_numpy():
    """Quotients of the shapes the assembly produces equal numpy's IEEE division."""
    import torch

    import paper_1305_3122_b200 as fa

    rng = np.random.default_rng(0)
    areas = np.concatenate([rng.uniform(1e-12, 1.0, 10000), [1e-300 * 1.5, 2.5e-300, 1.0, 3.0, 1e300]])
    kg = fa.batch_kg_mass(areas)
    assert np.array_equal(kg[0], areas / 6.0) and np.array_equal(kg[1], areas / 12.0)
