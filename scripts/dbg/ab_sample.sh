#!/bin/bash
# A/B of library variants on the C2 sampling call (graph mode, BPT_TRACE expand/compact times)
for v in "" "$@"; do
  echo "== ${v:-default}"
  BPT_LIB=$v BPT_TRACE=1 timeout 300 python scripts/phase_times.py --config C2 --reps 2 2>&1 | grep -E "sample \(graph\)|ms_median" | tail -2
done
