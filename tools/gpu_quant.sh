python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python bench.py --workload quantiles_gpt2_xl --steps 20 --warmup 3 > gpurun_out/bench_quant.json 2> gpurun_out/bench_quant.err; echo bench $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:quantiles --csv --log-file gpurun_out/launches_quant.csv python bench.py --workload quantiles_gpt2_xl --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sram_quantiles -s 1 -c 1 -o gpurun_out/quant_full python bench.py --workload quantiles_gpt2_xl --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_quant.log 2>&1; echo ncu2 $?
