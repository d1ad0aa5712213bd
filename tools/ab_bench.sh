#!/bin/bash
# usage: tools/ab_bench.sh "<env assignments>" lib1 lib2 ...  -> alternating sustained bench runs (200 steps)
envs="$1"; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo -n "$(basename $lib) $envs "; env $envs Q8_LIB_PATH=$lib python bench.py --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print(round(d['ms_per_step'],3),'ms', round(100*d['roofline']['frac'],1),'%', c['sm_mhz'],'MHz')"
  done
done
