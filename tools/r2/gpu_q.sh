#!/bin/bash
mkdir -p gpurun_out/r2
O=gpurun_out/r2
timeout 300 python tools/r2/xp_check.py check > $O/xp_check.log 2>&1; echo "rc=$?" >> $O/xp_check.log
tail -40 $O/xp_check.log
if grep -q "rc=0" $O/xp_check.log; then
timeout 300 python tools/r2/xp_check.py time 4096x4096x4096 8192x8192x8192 16384x16384x16384 4096x4096x65536 > $O/xp_time.log 2>&1
cat $O/xp_time.log
fi
