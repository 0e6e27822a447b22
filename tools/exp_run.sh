python -m pytest tests -m gpu -x -q > gpurun_out/e14_pytest.log 2>&1
tail -3 gpurun_out/e14_pytest.log
python bench.py --steps 5 --no-cpu-baseline > gpurun_out/e14_c2.json 2>gpurun_out/e14_c2.err
python bench.py --config 3 --no-cpu-baseline --steps 5 > gpurun_out/e14_c3.json 2>gpurun_out/e14_c3.err
