python tools/sweep.py 5 'LR_SPMV_HEAD=8192' 'LR_SPMV_HEAD=12288' 'LR_SPMV_HEAD=4096' > gpurun_out/e13_c5.txt 2>&1
