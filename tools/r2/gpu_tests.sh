#!/bin/bash
# pytest -m gpu + smoke on one B200; logs under gpurun_out/r2/
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 2400 python -m pytest tests -q -m gpu -x ${PYTEST_ARGS:-} > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log
