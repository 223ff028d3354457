#!/bin/bash
# SASS mnemonic census of every kernel in the product library (proves the
# tcgen05 / TMA / TMEM path: UTCHMMA, UTMALDG, UTMASTG, LDTM, STTM; no HMMA).
# usage: bash scripts/sass_census.sh [lib.so] > profiles/r02/sass_census.txt
lib=${1:-paper_2603_01960_b200/_lib/libtileattn_b200.so}
echo "# cuobjdump -sass $lib ($(date -u +%F), nvcc $(nvcc --version | grep -o 'V[0-9.]*'))"
cuobjdump -sass "$lib" | awk '
  /Function :/ { fn=$3; next }
  fn != "" && /\/\*[0-9a-f]{4,}\*\// {
    line=$0; sub(/.*\*\/ +/, "", line); split(line, t, /[ ;]/); op=t[1];
    if (op ~ /^@/) op=t[2]; sub(/\..*/, "", op); cnt[fn, op]++; fns[fn]=1 }
  END {
    n=split("UTCHMMA UTMALDG UTMASTG LDTM STTM MUFU FFMA2 FADD2 F2FP HMMA USETMAXREG SYNCS BAR LDL STL", ops, " ");
    printf "%-16s", "kernel"; for (i=1;i<=n;i++) printf " %8s", ops[i]; printf "\n";
    for (f in fns) { name=f; gsub(/_ZN2ta[0-9A-Za-z_]*sdpa_fwd_kernelI/, "sdpa<", name); name=substr(name,1,60);
      printf "%s\n%-16s", name, ""; for (i=1;i<=n;i++) printf " %8d", cnt[f, ops[i]]; printf "\n" } }'
