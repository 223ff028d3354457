"""SASS mnemonic census per kernel of the product library (tcgen05 / TMA /
TMEM evidence: UTCHMMA, UTMALDG, UTMASTG, LDTM, STTM; no HMMA).
usage: python scripts/sass_census.py [lib.so] > profiles/r02/sass_census.txt"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2603_01960_b200/_lib/libtileattn_b200.so"
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
OPS = ["UTCHMMA", "UTMALDG", "UTMASTG", "UTMACCTL", "LDTM", "STTM", "MUFU", "FFMA2", "FADD2",
       "F2FP", "HMMA", "USETMAXREG", "SYNCS", "BAR", "LDL", "STL"]
funcs, cur = {}, None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = funcs.setdefault(m.group(1), Counter())
        continue
    m = re.match(r"\s*/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
    if m and cur is not None:
        cur[m.group(2)] += 1
ver = subprocess.run(["nvcc", "--version"], capture_output=True, text=True).stdout.split()[-1]
print(f"# cuobjdump -sass {lib}; nvcc {ver}")
print(f"# kernel template args: <D, bf16, trace, Q tiles per CTA, keys per K/V tile>")
print(f"{'kernel':34s} " + " ".join(f"{o:>8s}" for o in OPS))
for name, c in sorted(funcs.items()):
    m = re.search(r"sdpa_fwd_kernelILi(\d+)ELb(\d)ELb(\d)ELi(\d)ELi(\d+)E", name)
    short = (f"sdpa_fwd<{m.group(1)},{'bf16' if m.group(2) == '1' else 'f16'},"
             f"{'trace' if m.group(3) == '1' else '-'},{m.group(4)},{m.group(5)}>") if m else \
        re.sub(r"_ZN2ta\w*?cu_\w{8}\d+", "", name)[:34]
    print(f"{short:34s} " + " ".join(f"{c[o]:8d}" for o in OPS))
