#!/bin/bash
mkdir -p gpurun_out/r2
BNN_LIB_PATH=$PWD/build/variants/libQ.so timeout 120 python tools/r2/sconv_repro.py > gpurun_out/r2/q.log 2>&1
grep -a "SCONV\|ok\|Error" gpurun_out/r2/q.log | head
