"""Per-kernel SASS instruction census of libraftgp.so (cuobjdump -sass): the tcgen05 / TMEM / bulk-copy / mbarrier
instructions that prove which kernels use the Blackwell paths (B200_PROFILING.md's SASS mnemonics), plus the
instruction count and register-heavy ops of every kernel. Writes a markdown table.

usage: python tools/sass_census.py [lib.so] > profiles/r02/sass_census.md"""
import collections
import re
import subprocess
import sys

KEYS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTCATOMSWS", "LDTM", "STTM", "UBLKCP", "UTMALDG", "UTMASTG", "SYNCS",
        "HMMA", "FFMA", "DFMA", "DADD", "IMAD", "MUFU", "ATOMS", "ATOMG", "RED", "LDG", "STG", "LDS", "STS", "SHFL"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.splitlines()
    return out if len(out) == len(names) else names


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2312_01560_b200/libraftgp.so"
    txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    funcs = collections.OrderedDict()
    cur = None
    for line in txt.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m:
            funcs[cur]["_total"] += 1
            op = m.group(1)
            for k in KEYS:
                if op == k or op.startswith(k):
                    funcs[cur][k] += 1
                    break
    names = demangle(list(funcs))
    print(f"# SASS census of `{lib}` (cuobjdump -sass; sm_100a)\n")
    print("Kernels that use the tcgen05 tensor cores (UTCHMMA = tcgen05.mma, LDTM = tcgen05.ld, UTCBAR = "
          "tcgen05.commit), bulk async copies (UBLKCP = cp.async.bulk) and mbarriers (SYNCS):\n")
    cols = ["UTCHMMA", "UTCBAR", "LDTM", "STTM", "UBLKCP", "UTMALDG", "SYNCS", "_total"]
    print("| kernel | " + " | ".join(c.strip("_") for c in cols) + " |")
    print("|---" * (len(cols) + 1) + "|")
    tc = [(n, c) for n, c in zip(names, funcs.values()) if c["UTCHMMA"] or c["LDTM"] or c["UBLKCP"]]
    for n, c in tc:
        print(f"| `{n[:110]}` | " + " | ".join(str(c[k]) for k in cols) + " |")
    print("\nEvery kernel (instruction counts by class):\n")
    cols2 = ["_total", "FFMA", "IMAD", "MUFU", "DFMA", "DADD", "ATOMS", "ATOMG", "RED", "LDG", "STG", "LDS", "STS", "SHFL"]
    print("| kernel | " + " | ".join(c.strip("_") for c in cols2) + " |")
    print("|---" * (len(cols2) + 1) + "|")
    for n, c in sorted(zip(names, funcs.values()), key=lambda x: x[0]):
        print(f"| `{n[:110]}` | " + " | ".join(str(c[k]) for k in cols2) + " |")


if __name__ == "__main__":
    main()
