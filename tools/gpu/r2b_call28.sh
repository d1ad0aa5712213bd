# LARS norms pass grid size: 1x / 2x / 4x the resident CTA slots (Q8_LARS_GRID_MULT), ABBA-style repeats.
O=gpurun_out/r2b28; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_layerwise.py -m gpu -q -p no:cacheprovider -k lars > $O/pytest.log 2>&1; echo pytest $?
for rep in 1 2 3; do for m in 1 2 4 1; do
  echo -n "mult $m "; Q8_LARS_GRID_MULT=$m timeout 300 python bench.py --workload lars_resnet50 --steps 30 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1e3,2),'us', round(d['roofline']['frac'],4))"
done; done > $O/grid.txt 2>&1; cat $O/grid.txt
for m in 1 2 4; do Q8_LARS_GRID_MULT=$m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/l$m.csv python bench.py --workload lars_resnet50 --steps 2 --warmup 2 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "mult $m: $(grep lars_norms $O/l$m.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"; done
