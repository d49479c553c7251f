"""Per-kernel SASS instruction census of libsketch_b200.so (cuobjdump): proof of tcgen05 / TMA / TMEM
use.  python tools/sass_census.py > profiles/r2_sass_census.txt"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTCHMMA", "UTCQMMA", "DMMA", "UTCBAR", "UTMALDG", "UBLKCP", "UTMASTG", "LDTM", "STTM", "SYNCS", "LDGSTS", "DADD",
        "DFMA", "FFMA", "LDS", "STS", "REDG", "BRX"]


def main():
    lib = os.path.join(ROOT, "paper_2508_21189_b200", "lib", "libsketch_b200.so")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    cur, counts = None, {}
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = {k: 0 for k in KEYS}
            continue
        if cur is None or not re.search(r"/\*[0-9a-f]{4,}\*/", line):
            continue
        ins = re.sub(r".*\*/\s*", "", line.split(";")[0]).strip()
        op = ins.split()[0] if ins else ""
        if op.startswith("@"):
            op = ins.split()[1]
        base = op.split(".")[0]
        for k in KEYS:
            if base == k:
                counts[cur][k] += 1
    names = sorted(counts)
    demangle = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
    print("# SASS census of paper_2508_21189_b200/lib/libsketch_b200.so (cuobjdump -sass; static instruction counts)")
    print("# " + " ".join(f"{k:>7s}" for k in KEYS) + "  kernel")
    for n, dn in zip(names, demangle):
        c = counts[n]
        if not any(c.values()):
            continue
        dn = re.sub(r"skb::\(anonymous namespace\)::", "", dn)[:110]
        print("  " + " ".join(f"{c[k]:7d}" for k in KEYS) + "  " + dn)


if __name__ == "__main__":
    sys.exit(main())
