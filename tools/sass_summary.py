"""Per-kernel SASS opcode summary of libdmt.so (tcgen05 / TMA evidence):
    python tools/sass_summary.py [libdmt.so] > profiles/<tag>_sass_opcodes.txt
Counts UTCHMMA / UTCQMMA (tcgen05.mma), UTMALDG (TMA loads), UBLKCP (bulk
copies), LDTM / STTM (TMEM ld/st), UTCBAR (tcgen05.commit) per function."""
import collections
import re
import subprocess
import sys

OPS = ["UTCHMMA", "UTCQMMA", "UTCIMMA", "UTMALDG", "UTMAPF", "UBLKCP", "LDTM", "STTM", "UTCBAR", "HMMA"]


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2403_00877_b200/libdmt.so"
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    fn, counts = None, collections.OrderedDict()
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            fn = m.group(1)
            counts[fn] = collections.Counter()
            continue
        if fn is None:
            continue
        for op in OPS:
            if re.search(r"\b" + op + r"\b", line):
                counts[fn][op] += 1
    demangle = {}
    try:
        names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout
        demangle = dict(zip(counts, names.splitlines()))
    except Exception:
        pass
    print(f"# SASS opcode counts per kernel ({lib}; cuobjdump -sass)")
    print("# " + " ".join(OPS))
    for f, c in counts.items():
        if not any(c.values()):
            continue
        print(" ".join(f"{op}={c[op]}" for op in OPS if c[op]), "|", demangle.get(f, f)[:200])


if __name__ == "__main__":
    main()
