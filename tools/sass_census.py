"""Per-kernel census of the Blackwell-native instructions in the built library (cuobjdump -sass):
tcgen05.mma -> UTCHMMA (kind::f16/tf32: UTCHMMA / UTCQMMA ...), tcgen05.ld/st -> LDTM/STTM, TMA tensor
loads -> UTMALDG, bulk copies -> UBLKCP, tcgen05.commit -> UTCBAR, TMEM alloc -> UTCATOMSWS.
usage: python tools/sass_census.py [lib.so] [out.md]"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1311_1419_b200", "_lib", "libcsenc.so")
out = sys.argv[2] if len(sys.argv) > 2 else None
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
KEYS = ["UTCHMMA", "UTCQMMA", "UTCIMMA", "UTCBAR", "LDTM", "STTM", "UTMALDG", "UTMAPF", "UBLKCP", "UTCATOMSWS", "SYNCS"]
per = collections.OrderedDict()
cur = None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        per[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    m = re.search(r"/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m:
        op = m.group(1)
        per[cur]["_instr"] += 1
        for k in KEYS:
            if op.startswith(k):
                per[cur][k] += 1


def short(n):
    d = subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip()
    d = re.sub(r"std::conditional<.*?>::type", "params", d)
    return d[:110]


rows = ["| kernel | SASS instr | " + " | ".join(KEYS) + " |", "|---|---|" + "---|" * len(KEYS)]
for n, c in per.items():
    rows.append(f"| `{short(n)}` | {c['_instr']} | " + " | ".join(str(c[k]) for k in KEYS) + " |")
text = (f"# SASS census of `{os.path.relpath(lib, ROOT)}` (cuobjdump -sass; tools/sass_census.py)\n\n"
        "tcgen05.mma -> UTCHMMA, tcgen05.commit -> UTCBAR, tcgen05.ld/st -> LDTM/STTM, TMA tensor load -> UTMALDG,\n"
        "TMA prefetch -> UTMAPF, cp.async.bulk -> UBLKCP, tcgen05.alloc -> UTCATOMSWS, mbarrier ops -> SYNCS.\n\n"
        + "\n".join(rows) + "\n")
if out:
    with open(out, "w") as f:
        f.write(text)
print(text)
