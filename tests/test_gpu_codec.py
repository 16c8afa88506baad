"""SURVEY.md sec. 8(f) row f4 on the GPU: the sec. 2 packetisation fused with
the exponentiation (text -> packets -> C, and C -> M -> text), parity with the
oracle's codec + modexp and the paper's worked example."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import oracle  # noqa: E402
import workload  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def R():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1407_1465_b200 as R
    return R


def test_paper_example_fused(R):
    g = json.load(open(os.path.join(GOLD, "sec2_packets.json")))
    dv = json.load(open(os.path.join(GOLD, "survey_derived.json")))
    c = R.rsa_encrypt_text(g["text"], g["e"], g["n"], 15)
    assert [int(v) for v in c.cpu().numpy().view(np.uint32).ravel()] == dv["toy_ciphertexts"]
    txt = R.rsa_decrypt_text(c, dv["toy_d"], g["n"], 15)
    assert bytes(txt.cpu().numpy()).decode() == g["decoded"]


@pytest.mark.parametrize("key,nbits", [("toy17947", 15), ("table2_513581", 19), ("rsa64", 64)])
def test_random_text_roundtrip(R, key, nbits):
    k = workload.key(key)
    rng = np.random.default_rng(nbits)
    letters = (rng.integers(0, 26, 2 * 300001) + ord("a")).astype(np.uint8)
    text = torch.from_numpy(letters).cuda()
    st = torch.full((300001,), 99, dtype=torch.int32, device="cuda")
    c = R.rsa_encrypt_text(text, k["e"], k["n"], nbits, status=st)
    torch.cuda.synchronize()
    assert int(st.abs().max()) == 0
    s = workload.limbs_needed(nbits)
    pk = np.array(oracle.encode(bytes(letters[:4000]).decode()), dtype=np.uint32).reshape(-1, 1)
    want = oracle.modexp_batch(pk, k["e"], k["n"])
    assert np.array_equal(c.cpu().numpy().view(np.uint32)[:2000], want[:, :s])
    back = R.rsa_decrypt_text(c, k["d"], k["n"], nbits, status=st)
    torch.cuda.synchronize()
    assert np.array_equal(back.cpu().numpy(), letters) and int(st.abs().max()) == 0


def test_codec_status(R):
    n, e = 17947, 131
    text = torch.tensor(list(b"paRa11el"), dtype=torch.uint8, device="cuda")
    st = torch.zeros(4, dtype=torch.int32, device="cuda")
    c = R.rsa_encrypt_text(text, e, n, 15, status=st)
    torch.cuda.synchronize()
    assert st.cpu().tolist() == [0, -7, -7, 0]
    # decrypting with the paper's invalid d = 137 (reading Z1): results that are
    # not packets come back as '??' with RSA_EPACKET, exactly where the oracle says
    good = R.rsa_encrypt_text("parallelencryption", e, n, 15)
    st9 = torch.zeros(9, dtype=torch.int32, device="cuda")
    txt = bytes(R.rsa_decrypt_text(good, 137, n, 15, status=st9).cpu().numpy()).decode()
    cvals = good.cpu().numpy().view(np.uint32).ravel()
    for i, cv in enumerate(cvals):
        m = oracle.modexp(int(cv), 137, n)
        ok = m // 100 <= 25 and m % 100 <= 25
        assert (st9[i].item() == 0) == ok
        assert txt[2 * i:2 * i + 2] == (oracle.decode([m]) if ok else "??")
    with pytest.raises(R.RsaError) as ei:
        R.rsa_encrypt_text("abc", e, n, 15)
    assert ei.value.code == R.RSA_EODD
    with pytest.raises(R.RsaError) as ei:
        R.rsa_encrypt_text("ab", 7, 187, 8)          # n = 187 cannot carry packets up to 2525
    assert ei.value.code == R.RSA_ERANGE
