#!/bin/bash
# usage: tools/ab.sh "<probe args>" lib1 lib2 ...   -> alternating probe runs (same box, same process env)
args="$1"; shift
for rep in 1 2; do
  for lib in "$@"; do
    echo -n "$(basename $lib) "; Q8_LIB_PATH=$lib python tools/probe_step.py $args | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms'],3),'ms', round(d['frac']*100,1),'%')"
  done
done
