#!/bin/bash
# usage: tools/ab_work.sh "<workloads>" steps lib1 lib2 [reps]  -> bench runs of each workload with each library
# (Q8_LIB_PATH), the library order reversed on every other repetition (ABBA: a power-capped box runs hotter
# on later runs); ms/step and roofline fraction per run
wls="$1"; steps="$2"; a="$3"; b="$4"; reps="${5:-4}"
for rep in $(seq 1 $reps); do
  if [ $((rep % 2)) -eq 1 ]; then order="$a $b"; else order="$b $a"; fi
  for w in $wls; do
    for lib in $order; do
      echo -n "$w $(basename $lib) "; Q8_LIB_PATH=$lib timeout 300 python bench.py --workload $w --steps $steps --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print(round(d['ms_per_step']*1e3,2),'us', round(d['roofline']['frac'],4), c['sm_mhz'],'MHz')"
    done
  done
done
