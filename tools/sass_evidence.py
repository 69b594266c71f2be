"""SASS evidence that the hot kernels are Blackwell-native (B200_PROFILING.md table).

    python tools/sass_evidence.py [lib.so] > profiles/r02_sass_opcodes.md

Static counts, per kernel of libsamp_b200.so, of the instructions that prove the path:
UTCIMMA / UTCHMMA (tcgen05.mma kind::i8 / kind::f16), UTMALDG (TMA tensor loads), LDTM /
STTM (tcgen05.ld / st), UTCBAR (tcgen05.commit) — and HMMA / IMMA (legacy mma.sync, must
be 0).  Runs on the build host (cuobjdump, no GPU).
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ("UTCIMMA", "UTCHMMA", "UTMALDG", "UTMASTG", "LDTM", "STTM", "UTCBAR", "HMMA", "IMMA", "FFMA2", "MUFU")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_2209_09130_b200", "lib", "libsamp_b200.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    counts = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur is None:
            continue
        m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and m.group(1) in OPS:
            counts[cur][m.group(1)] += 1
    names = {k: subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip() for k in counts}
    print("# SASS opcode evidence (static counts per kernel, libsamp_b200.so, sm_100a)\n")
    print("tcgen05.mma shows as UTCIMMA (kind::i8) / UTCHMMA (kind::f16), TMA as UTMALDG, tcgen05.ld/st as "
          "LDTM/STTM, tcgen05.commit as UTCBAR; legacy HMMA/IMMA must be absent.\n")
    print("| kernel | " + " | ".join(OPS) + " |")
    print("|---|" + "---|" * len(OPS))
    for k, c in counts.items():
        if not any(c[o] for o in OPS[:7]):
            continue
        short = re.sub(r"\(CUtensorMap_st.*", "", names[k]).replace("samp::", "")
        print(f"| `{short[:110]}` | " + " | ".join(str(c[o]) for o in OPS) + " |")
    tot = collections.Counter()
    for c in counts.values():
        tot.update(c)
    print(f"\nWhole library: HMMA {tot['HMMA']}, IMMA {tot['IMMA']}, UTCIMMA {tot['UTCIMMA']}, "
          f"UTCHMMA {tot['UTCHMMA']}, UTMALDG {tot['UTMALDG']}.")


if __name__ == "__main__":
    main()
