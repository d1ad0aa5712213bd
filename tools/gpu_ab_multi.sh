timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
for rep in 1 2; do for lib in paper_2110_02861_b200/libq8_base.so paper_2110_02861_b200/libq8.so; do
echo -n "cfg3 $(basename $lib) "; Q8_LIB_PATH=$lib python bench.py --workload cfg3_resnet50 --steps 200 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step']*1000,2),'us', round(100*d['roofline']['frac'],1),'%')"
done; done
bash tools/ab_layer.sh lamb_gpt2_xl paper_2110_02861_b200/libq8_base.so paper_2110_02861_b200/libq8.so
bash tools/ab.sh "--iters 20" paper_2110_02861_b200/libq8_base.so paper_2110_02861_b200/libq8.so
