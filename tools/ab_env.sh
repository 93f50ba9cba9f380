#!/bin/bash
# A/B of library builds on one index per config: bash tools/ab_env.sh "<configs>" <variant> [<variant> ...]
# variant "main" = in-tree libisax.so, else variants/<name>/libisax.so. Prints q/s, stage ms, counters.
cfgs=$1; shift
for c in $cfgs; do
  for v in "$@"; do
    if [ "$v" = main ]; then lib=""; else lib=variants/$v/libisax.so; fi
    ISAX_LIB=$lib timeout 300 python tools/sweep_env.py --config $c --var DUMMY --values 0 1 2>&1 | grep -v Warn | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    m=d['ms_first_round']
    print('cfg$c', '$v'.ljust(10), d['qps'], d['ms_step'], 'lbscan', m['lbscan'], 'cand', m['candcheck'], 'ref', m['refine'], 'win', m['window'], 'pairs', d['leaf_pairs_pq'], 'fb', d['first_band'])
"
  done
done
