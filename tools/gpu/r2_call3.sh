set -x
mkdir -p gpurun_out/r2
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo smoke $?
timeout 1500 python -m pytest tests -m gpu -q --durations=15 -p no:cacheprovider > gpurun_out/r2/pytest_all3.log 2>&1; echo pytest $?
tail -45 gpurun_out/r2/pytest_all3.log
