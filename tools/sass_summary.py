"""Per-kernel SASS census of libh2b.so: instruction count and the mnemonics
that show how each kernel moves and multiplies data (UBLKCP = TMA bulk
copy, DMMA = FP64 tensor-core MMA, DFMA = FP64 FMA, SYNCS = mbarrier ops,
ATOMG/REDG = global atomics).  Writes a table (profiles/r02_sass_summary.txt).

    python tools/sass_summary.py [--lib paper_1811_05731_b200/libh2b.so]
"""

import argparse
import re
import subprocess
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OPS = ["UBLKCP", "DMMA", "DFMA", "DADD", "DMUL", "SYNCS", "ATOMG", "REDG", "LDG", "STG", "LDS", "STS", "MEMBAR",
       "UTCMMA", "LDTM"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lib", default=str(ROOT / "paper_1811_05731_b200" / "libh2b.so"))
    ap.add_argument("--out", default=str(ROOT / "profiles" / "r02_sass_summary.txt"))
    a = ap.parse_args()
    sass = subprocess.run(["cuobjdump", "-sass", a.lib], capture_output=True, text=True, check=True).stdout
    funcs, cur = {}, None
    for line in sass.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)(\.[A-Z0-9_.]*)?", line)
        if m:
            funcs[cur]["_insts"] += 1
            op = m.group(1)
            for o in OPS:
                if op == o or op.startswith(o):
                    funcs[cur][o] += 1
    demangle = subprocess.run(["c++filt"], input="\n".join(funcs), capture_output=True, text=True).stdout.split("\n")
    rows = []
    for (mangled, cnt), name in zip(funcs.items(), demangle):
        short = re.sub(r"\(anonymous namespace\)::", "", name)
        short = re.sub(r"\(.*\)$", "", short)
        rows.append((short, cnt))
    hdr = f"{'kernel':<44} {'insts':>7} " + " ".join(f"{o:>7}" for o in OPS)
    lines = [f"SASS census of {Path(a.lib).name} (cuobjdump -sass; sm_100a)", hdr]
    for short, cnt in sorted(rows):
        lines.append(f"{short[:44]:<44} {cnt['_insts']:>7} " + " ".join(f"{cnt[o]:>7}" for o in OPS))
    Path(a.out).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
