# scratch driver for gpurun experiments (tools/build_variant.sh builds A/B libraries)
timeout 900 python -m pytest tests -m gpu -x -q
