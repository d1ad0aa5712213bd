# Re-entry sanity on a fresh box: smoke, GPU tests, default bench, cfg3/LARS lines.
O=gpurun_out/r2b1; mkdir -p $O
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $O/smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1; echo pytest $?
tail -3 $O/pytest_gpu.log
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_cfg4.json 2> $O/bench_cfg4.err; echo b1 $?
for w in cfg3_resnet50 lars_resnet50; do
  timeout 600 python bench.py --workload $w --steps 30 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; echo $w $?
done
cat $O/*.json | cut -c1-400
