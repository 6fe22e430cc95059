"""The device generator (tc_synth_*) produces exactly the numpy generator's words."""
import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a GPU", allow_module_level=True)

from paper_2605_17821_b200 import tc  # noqa: E402
from tests.gpu_util import to_np  # noqa: E402


@pytest.mark.parametrize("wb", [2, 4])
@pytest.mark.parametrize("structure", [synth.S1_IID, synth.S2_RUNS])
def test_device_generator_matches_numpy(wb, structure):
    n, start, seed, seg = 100003, 123456789, synth.SEED0 + 3, 2
    dt = torch.int16 if wb == 2 else torch.int32
    t = torch.empty(n, dtype=dt, device="cuda")
    tc.synth_base(t, seed, seg, start)
    exp = synth.base(n, wb, seed, seg, start)
    assert np.array_equal(to_np(t), exp)
    for v, f in ((1, 0.01), (2, 0.5), (3, 1.0)):
        tc.synth_step(t, seed, seg, v, synth.p53_of(f), structure, start)
        exp = synth.step(exp, seed, seg, v, f, structure, start)
        assert np.array_equal(to_np(t), exp)
