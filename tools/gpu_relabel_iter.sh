timeout 600 python -m pytest tests -q -m gpu -x -k "relabel or grey or cluster or near_tie or config4_prefix" > gpurun_out/it2_tests.log 2>&1; echo "rc=$?" >> gpurun_out/it2_tests.log
CMD="python tools/run_cfg.py 4 1e7" bash tools/gpu_variants.sh
