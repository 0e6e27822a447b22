python -m pytest tests -m gpu -x -q > gpurun_out/e4_pytest.log 2>&1
tail -1 gpurun_out/e4_pytest.log
python bench.py --no-cpu-baseline --steps 5 > gpurun_out/e4_c2.json 2>/dev/null
python bench.py --config 3 --no-cpu-baseline --steps 5 > gpurun_out/e4_c3.json 2>/dev/null
