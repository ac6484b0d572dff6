#!/bin/bash
timeout 600 python -m pytest -q -x tests/test_gpu_signpack.py -k small_channel 2>&1 | tail -2
timeout 300 python tools/r2/sconv_hang.py 2>&1 | grep -v "^blk" | tail -2
timeout 120 python tools/r2/sconv_timeline.py 0 0 2>&1 | head -10
timeout 300 python tools/r2/sconv_ablate.py
