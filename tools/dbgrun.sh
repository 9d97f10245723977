python -m pytest tests/test_gpu_msed_tc.py -x -q 2>&1 | tail -2
bash tools/launches.sh | grep msed_tc
