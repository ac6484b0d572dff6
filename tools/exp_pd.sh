python tools/pack_only.py >> gpurun_out/exp_pd.log 2>&1
BNN_PACK_PIX=64 python tools/pack_only.py 2>&1 | head -1 >> gpurun_out/exp_pd.log
