# scratch experiment driver (gpurun): K4c vs K4b, head sweep
python -m pytest tests -m gpu -x -q > gpurun_out/e2_pytest.log 2>&1
tail -3 gpurun_out/e2_pytest.log
LR_SPMV=tile python bench.py --no-cpu-baseline --steps 5 > gpurun_out/e2_c2_tile.json 2>/dev/null
for h in 8192 12288 16384; do
  LR_SPMV_HEAD=$h python bench.py --no-cpu-baseline --steps 5 > gpurun_out/e2_c2_seg$h.json 2>gpurun_out/e2_c2_seg$h.err
done
LR_SPMV=tile python bench.py --config 3 --no-cpu-baseline --steps 5 > gpurun_out/e2_c3_tile.json 2>/dev/null
python bench.py --config 3 --no-cpu-baseline --steps 5 > gpurun_out/e2_c3_seg.json 2>/dev/null
