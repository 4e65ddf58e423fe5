"""z-vote ground filter through the C ABI vs the oracle (O9):
keep mask and counts bit-exact (integer work on an fp32 decision taken the same
way on both sides)."""
import numpy as np
import pytest

import gen

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2308_07173_b200 as g  # noqa: E402

DEV = torch.device("cuda:0")


def D(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("cell,mc", [(0.5, 10), (0.2, 3), (1.0, 1)])
def test_ground_filter_bitwise(orc, cell, mc):
    sc, _ = gen.scan(100_000, 150.0, 77)  # vehicle frame, banked ground + walls + posts
    keep, cnt = g.ground_filter(D(sc), cell, mc, with_count=True)
    ok, oc = orc.ground_filter(sc, cell, mc)
    assert np.array_equal(cnt.cpu().numpy(), oc)
    assert np.array_equal(keep.cpu().numpy(), ok)


def test_ground_filter_edges(orc):
    # points exactly on cell boundaries and negative coordinates
    ij = np.stack(np.meshgrid(np.arange(-20, 20), np.arange(-20, 20)), -1).reshape(-1, 2) * 0.5
    p = np.column_stack([np.repeat(ij, 3, axis=0), np.tile([0.0, 1.0, 2.0], len(ij))]).astype(np.float32)
    keep, cnt = g.ground_filter(D(p), 0.5, 3, with_count=True)
    ok, oc = orc.ground_filter(p, 0.5, 3)
    assert np.array_equal(cnt.cpu().numpy(), oc) and np.array_equal(keep.cpu().numpy(), ok)
    assert g.ground_filter(torch.zeros((0, 3), dtype=torch.float32, device=DEV), 0.5, 3).numel() == 0
    with pytest.raises(g.GicpError):
        g.ground_filter(D(p), 0.0, 3)
