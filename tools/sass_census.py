"""SASS instruction census of the in-tree library: per kernel, the counts of the mnemonics that
prove the tensor-core / TMA / TMEM path (B200_PROFILING.md: UTCHMMA/UTCQMMA = tcgen05.mma,
UTMALDG/UBLKCP = TMA tensor / bulk copies, LDTM/STTM = tcgen05.ld/st, UTCBAR = tcgen05.commit),
plus the packed fp32 and local-memory (spill) instructions. Usage:
    python tools/sass_census.py [lib.so] > profiles/sass_census_rNN.md"""
import collections
import re
import subprocess
import sys

MNEMS = ["UTCHMMA", "UTCQMMA", "UTCBAR", "UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "LDTM", "STTM",
         "FFMA2", "FADD2", "FMUL2", "HMMA", "LDL", "STL", "SYNCS", "BAR", "ATOMG", "RED"]


def demangle(names):
    out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout
    return out.strip().split("\n")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2112_13509_b200/libautobyte.so"
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    kernels = collections.OrderedDict()
    cur = None
    for line in sass.split("\n"):
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            kernels[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?", line)
        if m:
            kernels[cur]["_total"] += 1
            op = m.group(1)
            if op in MNEMS:
                kernels[cur][op] += 1
    names = demangle(list(kernels))
    cols = [c for c in MNEMS if any(k[c] for k in kernels.values())]
    print(f"# SASS census of `{lib}` (cuobjdump -sass, sm_100a)\n")
    print("| kernel | instrs | " + " | ".join(cols) + " |")
    print("|---|---:|" + "---:|" * len(cols))
    for (mangled, cnt), name in zip(kernels.items(), names):
        name = name.replace("ab::", "").split("(")[0]
        print(f"| `{name}` | {cnt['_total']} | " + " | ".join(str(cnt[c]) for c in cols) + " |")


if __name__ == "__main__":
    main()
