# AdamW8bit.step() over GPT-2-XL's 580 tensors (plan, 2 launches) vs the flat kernel: ncu summaries.
O=gpurun_out/r2b23; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:optim8bit_step -s 10 -c 2 -o /tmp/api_full python bench.py --workload optim_api_gpt2_xl --steps 2 --warmup 5 --no-cpu-baseline --no-e2e > /dev/null 2>&1; echo ncu $?
python tools/ncu_metrics.py /tmp/api_full.ncu-rep > $O/ncu_api.txt 2>&1
grep -E "==|gpu__time|inst_executed.sum |issue_active|dram__bytes|stalls|registers|wavefronts_mem_shared.sum" $O/ncu_api.txt
ncu -i /tmp/api_full.ncu-rep --page source --csv --print-source sass > $O/api_source.csv 2>/dev/null; echo src $?
