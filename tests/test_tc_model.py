"""Design check, on CPU, of the CUDA-core half of the tensor-core Montgomery
multiply (paper_1407_1465_b200/csrc/tc_digits.cuh, modexp_tc.cu): the product
T = A B streamed out as 32-bit words (rolled row form mul_rows, the column
scans sqr_scan / sqr_col) and the word <-> 52-bit digit
conversions, compiled for the host (tests/tools/tc_model.cu, rounding toward
zero) and compared with Python integers.  The reduction half runs on the
tensor core and is pinned on the GPU (tests/test_gpu_shapes.py, and the whole
parity suite runs through it: the 2048-bit class defaults to it)."""
import os
import random
import shutil
import subprocess

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "tools", "tc_model.cu")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.fixture(scope="module")
def model(tmp_path_factory):
    if not os.path.exists(NVCC) and not shutil.which("nvcc"):
        pytest.skip("nvcc not available")
    exe = str(tmp_path_factory.mktemp("tc") / "tc_model")
    subprocess.check_call([NVCC, "-O2", "-std=c++17", "-o", exe, SRC])
    p = subprocess.Popen([exe], stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)

    def call(line):
        p.stdin.write(line + "\n")
        p.stdin.flush()
        return int(p.stdout.readline().strip(), 16)
    yield call
    p.stdin.close()
    p.wait()


def operands(rng):
    """Random 2048-bit operands and the structured extremes (all-ones digits,
    single bits at the 52/32-bit boundaries, zero, the maximum 2^2048 - 1)."""
    top = (1 << 2048) - 1
    fixed = [(top, top), (0, top), (1, 1), (top, 1), (1 << 2047, 1 << 2047), ((1 << 2080 - 1) & top, top),
             (int("f" * 13, 16) << 52 * 17, top), ((1 << 1040) - 1, (1 << 1040) - 1)]
    yield from fixed
    for _ in range(40):
        yield rng.getrandbits(2048), rng.getrandbits(2048)
    for _ in range(10):     # sparse operands: runs of zero digits and words
        a = sum(rng.getrandbits(52) << (52 * k) for k in rng.sample(range(39), 5))
        b = sum(((1 << 32) - 1) << (32 * k) for k in rng.sample(range(64), 7))
        yield a & top, b & top


def test_product_words(model):
    rng = random.Random(7)
    for a, b in operands(rng):
        assert model(f"M {a:x} {b:x}") == a * b


@pytest.mark.parametrize("op", ["Q", "R"])
def test_square_words(model, op):
    rng = random.Random(9)
    for a, _ in operands(rng):
        assert model(f"{op} {a:x}") == a * a


def test_product_split_rows(model):
    """mul_rows_f with NR < ND rows: the two row halves of one product, summed."""
    rng = random.Random(12)
    for a, b in operands(rng):
        assert model(f"P {a:x} {b:x}") == a * b


def test_square_words_1024(model):
    rng = random.Random(11)
    for a, _ in operands(rng):
        a &= (1 << 1024) - 1
        assert model(f"H {a:x}") == a * a


def test_words_digits_roundtrip(model):
    rng = random.Random(10)
    for a, _ in operands(rng):
        assert model(f"W {a:x}") == a


@pytest.mark.parametrize("op", ["E", "F"])
def test_runtime_word_emitter(model, op):
    """The 4096-bit kernel's run-time packer (digits leave a rolled loop as
    words), with branches (E) and branch-free (F, the kernel's default)."""
    rng = random.Random(13)
    for a, _ in operands(rng):
        assert model(f"{op} {a:x}") == a


@pytest.mark.parametrize("op", ["B", "C"])
def test_square_blocks(model, op):
    """sqr_blocks: the rolled block triangle (blocks of 10 / 8 digits at ND = 40)."""
    rng = random.Random(14)
    for a, _ in operands(rng):
        assert model(f"{op} {a:x}") == a * a


def test_square_blocks_4096(model):
    """sqr_blocks at the 4096-bit class's ND = 80 (the kernel's instance)."""
    rng = random.Random(15)
    top = (1 << 4096) - 1
    cases = [top, 0, 1, 1 << 4095, (1 << 4160 - 1) & top, int("f" * 13, 16) << 52 * 70]
    cases += [rng.getrandbits(4096) for _ in range(30)]
    cases += [sum(rng.getrandbits(52) << (52 * k) for k in rng.sample(range(78), 6)) & top for _ in range(10)]
    for a in cases:
        assert model(f"G {a:x}") == a * a


def test_product_blocks(model):
    """mul_blocks: the rolled block product at ND = 40."""
    rng = random.Random(16)
    for a, b in operands(rng):
        assert model(f"N {a:x} {b:x}") == a * b


def test_product_blocks_4096(model):
    """mul_blocks at ND = 80 with the kernel's slot aliasing (high digits over A)."""
    rng = random.Random(17)
    top = (1 << 4096) - 1
    cases = [(top, top), (0, top), (1, 1), (top, 1), (1 << 4095, 1 << 4095)]
    cases += [(rng.getrandbits(4096), rng.getrandbits(4096)) for _ in range(30)]
    cases += [(sum(rng.getrandbits(52) << (52 * k) for k in rng.sample(range(78), 6)) & top,
               sum(((1 << 32) - 1) << (32 * k) for k in rng.sample(range(128), 9))) for _ in range(10)]
    for a, b in cases:
        assert model(f"O {a:x} {b:x}") == a * b
