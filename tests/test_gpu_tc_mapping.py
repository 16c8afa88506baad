"""Work-mapping boundaries of the tensor-core kernels (modexp_tc.cu): one
packet, ragged 128-packet tile jobs (127/129), a partial trip with idle tiles,
and one persistent wave +- 1 (148 SMs x 256 at 2048 bits; the 1024-bit
instance's 4 tiles x 128, the 4096-bit instance's one tile), every output
element compared with the oracle (e = 65537 keeps the oracle fast; the op
list still covers squarings, the table-free multiply by g and the conversions)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import workload  # noqa: E402


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1407_1465_b200 as R
    return R


def _wave(R, key):
    k = workload.key(key)
    info = R.rsa_plan_info(k["e"], k["n"], k["nbits"])
    return info["grid"] * info["block"] if info["grid"] else 148 * 256


@pytest.mark.parametrize("key", ["rsa2048", "rsa1024", "rsa4096"])
def test_tc_mapping_boundaries(R, key):
    k = workload.key(key)
    nb = k["nbits"]
    s = workload.limbs_needed(nb)
    assert R.rsa_get_kernel_path(next(c for c in (32, 64, 128) if s <= c)) == R.RSA_PATH_TC
    wave = _wave(R, key)
    counts = [1, 127, 128, 129, 300, wave - 1, wave + 1]
    if key == "rsa2048":
        counts += [wave + 128 * 148 - 1]          # a trip whose jobs fill tile 0 of every CTA, minus one
    for count in counts:
        base = workload.packets(count, nb, n=k["n"], config_id=31)
        t = torch.from_numpy(base.view(np.int32)).cuda()
        got = R.rsa_modexp_batch(t, k["e"], k["n"], nb).cpu().numpy().view(np.uint32)
        want = oracle.modexp_batch(base, k["e"], k["n"])[:, :s]
        assert np.array_equal(got, want), (key, count)
