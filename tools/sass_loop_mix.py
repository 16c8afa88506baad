#!/usr/bin/env python3
"""Instruction mix of the hottest loops of a kernel in a cubin/.so/.o (SASS).

    python tools/sass_loop_mix.py <binary> <kernel-substring> [--top 3]

Finds backward branches (loops), prints each loop's size and opcode counts,
so a code change can be judged (IMAD.WIDE per product, IMAD.MOV on the FMA
pipe, shuffles) before spending GPU time."""
import re
import subprocess
import sys
from collections import Counter


def functions(binary):
    txt = subprocess.run(["cuobjdump", "-sass", binary], capture_output=True, text=True).stdout
    for f in re.split(r"\n\s+Function : ", txt)[1:]:
        name = f.split("\n")[0]
        ins = []
        for l in f.split("\n"):
            m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/\s+(.*?);", l)
            if m:
                ins.append((int(m.group(1), 16), m.group(2).strip()))
        yield name, ins


def op(text):
    t = text.split()
    return t[1] if t[0].startswith("@") else t[0]


def main():
    binary, pat = sys.argv[1], sys.argv[2]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 3
    for name, ins in functions(binary):
        if pat not in name:
            continue
        print(f"== {name}  ({len(ins)} instructions)")
        loops = []
        for a, t in ins:
            m = re.search(r"BRA(?:\.\w+)?\s+(?:\S+\s+)?0x([0-9a-f]+)", t)
            if m and int(m.group(1), 16) < a:
                lo = int(m.group(1), 16)
                body = [x for x in ins if lo <= x[0] <= a]
                loops.append((len(body), lo, a, body))
        sel = []
        for n, lo, hi, body in sorted(loops):
            c = Counter(op(t) for _, t in body)
            wide = c["IMAD.WIDE.U32"] + c["IMAD.WIDE.U32.X"]
            if wide >= 16:
                sel.append((n, lo, hi, c, wide))
        for n, lo, hi, c, wide in sel[:top]:
            print(f"  loop {lo:#x}-{hi:#x}: {n} instr, IMAD.WIDE* {wide}, IMAD.MOV {c['IMAD.MOV.U32']}, "
                  f"LOP3 {c['LOP3.LUT']}, MOV {c['MOV']}")
            print("   ", ", ".join(f"{k} {v}" for k, v in c.most_common(14)))


if __name__ == "__main__":
    main()
