#!/bin/bash
# usage: tools/ab_work.sh "<workloads>" steps lib1 lib2 ...  -> alternating bench runs of each workload with
# each library (Q8_LIB_PATH), 3 repetitions: ms/step and roofline fraction per run
wls="$1"; steps="$2"; shift 2
for rep in 1 2 3; do
  for w in $wls; do
    for lib in "$@"; do
      echo -n "$w $(basename $lib) "; Q8_LIB_PATH=$lib timeout 300 python bench.py --workload $w --steps $steps --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print(round(d['ms_per_step']*1e3,2),'us', round(d['roofline']['frac'],4), c['sm_mhz'],'MHz')"
    done
  done
done
