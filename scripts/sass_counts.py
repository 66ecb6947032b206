"""Opcode histogram per kernel from `cuobjdump -sass` of a cubin / .o / .so (no GPU needed).

    python scripts/sass_counts.py <file> [--filter SUBSTR] [--top N]

Prints, for every function whose mangled name contains SUBSTR, the count of each SASS opcode
(with modifiers, e.g. IMAD.WIDE.U32).  Used to check that the microbenchmarks time the
instruction they claim to (tests/test_abi.py) and to commit instruction mixes
(profiles/r02_sass_counts.txt)."""
import argparse
import collections
import re
import subprocess
import sys

OP = re.compile(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P[T0-9]+\s+)?([A-Z][A-Z0-9_]*(?:\.[A-Z0-9_]+)*)")


def counts(path, filt=""):
    out = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True, check=True).stdout
    res, cur = {}, None
    for ln in out.splitlines():
        if "Function :" in ln:
            name = ln.split("Function :", 1)[1].strip()
            cur = collections.Counter() if filt in name else None
            if cur is not None:
                res[name] = cur
            continue
        if cur is None:
            continue
        m = OP.search(ln)
        if m:
            cur[m.group(1)] += 1
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--filter", default="")
    ap.add_argument("--top", type=int, default=12)
    a = ap.parse_args()
    for name, c in counts(a.path, a.filter).items():
        tot = sum(c.values())
        print(f"{name}  ({tot} instructions)")
        print("   " + ", ".join(f"{k} {v}" for k, v in c.most_common(a.top)))


if __name__ == "__main__":
    sys.exit(main())
