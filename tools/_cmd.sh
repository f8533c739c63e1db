timeout 900 python -m pytest tests -m gpu -x -q -k "binning or order or tile" > gpurun_out/n14_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/n14_pytest.log
bash tools/ab.sh default
PROFILE_VIEWS=1 timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/c4z.csv python tools/profile_view.py > gpurun_out/c4z.log 2>&1; echo "c4 rc=$?"
