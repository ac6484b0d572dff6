mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "umma3 or variant or randomized or im2col" > gpurun_out/pytest_v3.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_v3.log
timeout 600 python tools/engine_contest.py > gpurun_out/contest.md 2>&1
