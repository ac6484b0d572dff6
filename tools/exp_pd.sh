BNN_UMMA_DEBUG=16 timeout 120 python tools/umma_stages_conv.py 2>&1 | grep -v "^ " > gpurun_out/stages_conv.log
timeout 300 python tools/race_check.py 5 > gpurun_out/race.log 2>&1
timeout 300 python bench.py --steps 20 --warmup 3 2>&1 | tail -1 > gpurun_out/bench_c2.json
