# cfg4 sustained (200 steps) under the power cap for the sub-block configurations of the bf16 step
# (Q8_NSUB x Q8_SUBT), two rounds in rotated order.
# (result: the default 4 x 128 is fastest under the cap too: 4.226 ms vs 4.43 (3 x 128, 3 x 256) and 4.84 (2 x 256))
O=gpurun_out/r2c10; mkdir -p $O
for rep in 1 2; do
  if [ $rep -eq 1 ]; then cfgs="4:128 3:128 2:256 3:256"; else cfgs="3:256 2:256 3:128 4:128"; fi
  for c in $cfgs; do
    ns=${c%%:*}; st=${c##*:}
    echo -n "nsub $ns subt $st: "
    Q8_NSUB=$ns Q8_SUBT=$st timeout 600 python bench.py --steps 200 --warmup 10 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); c=d['clocks']; print(round(d['ms_per_step'],4),'ms', round(d['roofline']['frac'],4), c['sm_mhz'],'MHz', c['reasons'], c.get('power_w_median'))"
  done
done
