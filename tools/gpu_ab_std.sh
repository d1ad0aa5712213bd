# standard A/B of paper_2110_02861_b200/libq8_base.so vs libq8.so: GPU tests, probes, sustained bench, cfg2/cfg3, LAMB
timeout 900 python -m pytest tests -m gpu -x -q -k "not exhaustive" 2>&1 | tail -1
bash tools/ab.sh "--iters 30" paper_2110_02861_b200/libq8_base.so paper_2110_02861_b200/libq8.so
bash tools/ab.sh "--iters 30 --kind momentum --gdt float16" paper_2110_02861_b200/libq8_base.so paper_2110_02861_b200/libq8.so
bash tools/ab_bench.sh "" paper_2110_02861_b200/libq8_base.so paper_2110_02861_b200/libq8.so
for rep in 1 2; do for lib in paper_2110_02861_b200/libq8_base.so paper_2110_02861_b200/libq8.so; do
echo -n "cfg2 $(basename $lib) "; Q8_LIB_PATH=$lib python bench.py --workload cfg2_gpt2_medium --steps 200 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4),'ms', round(100*d['roofline']['frac'],1),'%')"
echo -n "cfg3 $(basename $lib) "; Q8_LIB_PATH=$lib python bench.py --workload cfg3_resnet50 --steps 200 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2),'us', round(100*d['roofline']['frac'],1),'%')"
done; done
bash tools/ab_layer.sh lamb_gpt2_xl paper_2110_02861_b200/libq8_base.so paper_2110_02861_b200/libq8.so
