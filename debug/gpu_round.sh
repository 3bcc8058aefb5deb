set -x
timeout 900 python -m pytest tests/test_gpu_forward.py -x -q -k "engine" > gpurun_out/gt_engine.log 2>&1; echo engine=$?
timeout 900 python bench.py > gpurun_out/bench2.log 2>&1; echo bench=$?
tail -3 gpurun_out/gt_engine.log
