timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/n22_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/n22_pytest.log
bash tools/ab.sh default default
