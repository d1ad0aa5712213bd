# usage: tools/ab_layer.sh workload lib1 lib2 ...  -> alternating layer-wise bench runs
w="$1"; shift
for rep in 1 2; do for lib in "$@"; do
echo -n "$(basename $lib) "; Q8_LIB_PATH=$lib python bench.py --workload $w --steps 50 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3),'ms', round(100*d['roofline']['frac'],1),'%', d['clocks']['sm_mhz'])"
done; done
