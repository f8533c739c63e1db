timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/n9_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/n9_pytest.log
bash tools/ab.sh default g2 g1
