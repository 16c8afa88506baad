"""Check the tensor-core Montgomery reduction (csrc/microbench/tc_redc.cu) on a GPU box.

Writes in.bin (a random odd 2048-bit n, n' = -n^-1 mod 2^2048, T = A B with
A, B < n per packet), runs the binary, and checks U == T R^-1 mod n and the
quotient m == (T mod R) n' mod R with Python integers.
"""
from __future__ import annotations

import random
import struct
import subprocess
import sys

R = 1 << 2048


def main() -> int:
    exe = sys.argv[1]
    count = int(sys.argv[2]) if len(sys.argv) > 2 else 148 * 256
    reps = sys.argv[3] if len(sys.argv) > 3 else "1"
    rng = random.Random(1407)
    n = rng.getrandbits(2048) | (1 << 2047) | 1
    npr = (-pow(n, -1, R)) % R
    Ts = []
    for i in range(count):
        if i % 7 == 0:      # extremes: A, B = n - 1, 0, 1
            a = [n - 1, 0, 1, n - 1][i // 7 % 4]
            b = [n - 1, n - 1, 1, 1][i // 7 % 4]
            Ts.append(a * b)
        elif i % 7 == 3:
            # the subtraction's rare path: U' = (T + m n) / R placed at n - d, n or
            # n + d (top word equal to n's: the full borrow chain decides).  With
            # T = U' R - m n the kernel's own quotient (T mod R) n' mod R is m again.
            d = [0, 1, 2, 1 << 40, (1 << 200) + 5][i // 7 % 5]
            u = [n - d, n + d][i // 7 % 2] if d else n
            m = rng.randrange(R // 4, R // 2)
            Ts.append(u * R - m * n)
        else:
            a, b = rng.randrange(n), rng.randrange(n)
            Ts.append(a * b)
    assert all(0 <= t < n * R for t in Ts)
    with open("in.bin", "wb") as f:
        f.write(struct.pack("<i", count))
        f.write(n.to_bytes(256, "little"))
        f.write(npr.to_bytes(256, "little"))
        for t in Ts:
            f.write(t.to_bytes(512, "little"))
    r = subprocess.run([exe, "in.bin", "out.bin", reps], capture_output=True, text=True)
    print(r.stdout, r.stderr)
    if r.returncode:
        return r.returncode
    data = open("out.bin", "rb").read()
    rinv = pow(R, -1, n)
    bad_u = bad_m = 0
    for i, t in enumerate(Ts):
        u = int.from_bytes(data[256 * i:256 * (i + 1)], "little")
        m = int.from_bytes(data[256 * count + 256 * i:256 * count + 256 * (i + 1)], "little")
        if m != ((t % R) * npr) % R:
            bad_m += 1
            if bad_m < 3:
                em = ((t % R) * npr) % R
                diff = [k for k in range(256) if (m >> (8 * k)) & 255 != (em >> (8 * k)) & 255]
                print(f"pkt {i}: m differs at bytes {diff[:8]}..{diff[-4:]} ({len(diff)})")
        if u != (t * rinv) % n:
            bad_u += 1
            if bad_u < 3:
                eu = (t * rinv) % n
                print(f"pkt {i}: U differs; U-exp = {u - eu} (n multiple? {(u - eu) % n == 0})")
    print(f"checked {count}: bad_m {bad_m}, bad_u {bad_u}")
    return 0 if bad_m == 0 and bad_u == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
