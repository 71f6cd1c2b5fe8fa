"""Opcode histogram of every innermost loop body (backward branch) of one kernel's SASS.

    python tools/sass_loops.py paper_1902_09465_b200/libaknn.so k_advance_tiles

Used to check, without a GPU, how many fma-heavy-pipe instructions (IMAD*, IMAD.WIDE)
a hot loop spends per Philox block before measuring it."""
import collections
import re
import subprocess
import sys


def sass(lib, kernel):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    blocks = re.split(r"\n\s*Function : ", out)
    for b in blocks:
        name = b.split("\n", 1)[0].strip()
        if kernel in name:
            return name, b
    raise SystemExit(f"{kernel} not found")


def main():
    lib, kernel = sys.argv[1], sys.argv[2]
    name, body = sass(lib, kernel)
    ins = []
    for ln in body.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    print(name)
    for addr, txt in ins:
        m = re.search(r"BRA\s+(?:\w+\s*,\s*)?0x([0-9a-f]+)", txt)
        if not m:
            continue
        tgt = int(m.group(1), 16)
        if tgt >= addr:
            continue
        body_ins = [t for a, t in ins if tgt <= a <= addr]
        if len(body_ins) < 40:
            continue
        c = collections.Counter()
        for t in body_ins:
            op = t.split()[0]
            if op.startswith("@"):
                op = t.split()[1]
            parts = op.split(".")
            key = ".".join(parts[:2]) if parts[0] == "IMAD" else parts[0]
            c[key] += 1
        heavy = sum(v for k, v in c.items() if k.startswith("IMAD") or k in ("IDP",))
        print(f"loop 0x{tgt:x}-0x{addr:x}: {len(body_ins)} instrs, IMAD* {heavy}:",
              ", ".join(f"{k} {v}" for k, v in c.most_common(14)))


if __name__ == "__main__":
    main()
