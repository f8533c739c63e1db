timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r01l_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r01l_pytest.log
bash tools/gpu_round.sh r01l notests
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r01l_c5_bench.log 2>&1; echo "c5 rc=$?"; tail -1 gpurun_out/r01l_c5_bench.log | cut -c1-200
