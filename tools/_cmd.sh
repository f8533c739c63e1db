timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/n16_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/n16_pytest.log
bash tools/ab.sh default
PROFILE_VIEWS=1 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --profile-from-start off -k regex:k_project --csv --log-file gpurun_out/c4p2.csv python tools/profile_view.py > gpurun_out/c4p2.log 2>&1; echo "c4 rc=$?"
PROFILE_CONFIG=5 PROFILE_VIEWS=1 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --profile-from-start off -k regex:k_project --csv --log-file gpurun_out/c5p2.csv python tools/profile_view.py > gpurun_out/c5p2.log 2>&1; echo "c5 rc=$?"
