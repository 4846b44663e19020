#!/bin/bash
# SASS instruction histogram of the FAST kernels (evidence that the hot path
# runs tcgen05 / TMEM / bulk-copy instructions): per kernel, counts of the
# Blackwell tensor-core and async-copy opcodes plus the top opcodes overall.
#   tools/sass_histogram.sh > profiles/r02_sass_histogram.txt
set -e
cd "$(dirname "$0")/.."
for obj in build/sfg/sfg_mega.o build/sfg/sfg_fast.o build/sfg/sfg_attn.o build/sfg/sfg_attn_tc.o build/sfg/sfg_common.o; do
  echo "=== $obj"
  cuobjdump -sass "$obj" | awk '
    /Function :/ { fn = $3 }
    /^ *\/\*[0-9a-f]+\*\// {
      line = $0; sub(/^ *\/\*[0-9a-f]+\*\/ */, "", line); sub(/ *;.*/, "", line);
      split(line, t, " "); op = t[1]; if (op ~ /^@/) op = t[2];
      split(op, o, "."); base = o[1];
      cnt[fn "|" base]++; tot[fn]++
    }
    END {
      for (k in cnt) { split(k, p, "|"); if (p[2] ~ /^(UTCHMMA|UTCQMMA|UTCBAR|UTCATOMSWS|LDTM|STTM|UTCCP|UBLKCP|UBLKPF|SYNCS|UTMALDG|UTMASTG|HMMA|MEMBAR|FENCE|RED|ATOMG|BAR)$/) printf "%-60.60s %-12s %6d\n", p[1], p[2], cnt[k] }
      for (f in tot) printf "%-60.60s %-12s %6d\n", f, "(total)", tot[f]
    }' | sort
done
