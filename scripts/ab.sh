#!/bin/bash
# A/B timing of the default library and variants on C2 theta=8192: scripts/ab.sh [variant.so ...]
python scripts/sample_sweep.py --config C2 --theta 8192 --batches 1 --reps 2 2>&1 | grep '"rep": 1' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('default', round(d['s']*1e3,1), 'ms, expand', round(d['ms_expand'],1), 'coins', d['coins'])"
for v in "$@"; do
BPT_LIB=$v python scripts/sample_sweep.py --config C2 --theta 8192 --batches 1 --reps 2 2>&1 | grep '"rep": 1' | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', round(d['s']*1e3,1), 'ms, expand', round(d['ms_expand'],1), 'coins', d['coins'])"
done
