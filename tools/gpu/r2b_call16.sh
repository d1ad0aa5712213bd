# find_tensor next-tensor fast path: ABBA A/B of cfg3 (6 reps) and LAMB (4 reps).
O=gpurun_out/r2b16; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/ab_work.sh "cfg3_resnet50" 50 tools/ab/libq8_s3b.so tools/ab/libq8_new.so 6 > $O/ab_cfg3.txt 2>&1; cat $O/ab_cfg3.txt
bash tools/ab_work.sh "lamb_gpt2_xl" 20 tools/ab/libq8_s3b.so tools/ab/libq8_new.so 4 > $O/ab_lamb.txt 2>&1; cat $O/ab_lamb.txt
