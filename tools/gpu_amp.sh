set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_autocast.py tests/test_tnsr.py -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_amp.log
cat gpurun_out/pytest_amp.log
