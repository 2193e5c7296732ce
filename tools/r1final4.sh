# 4-GPU round-end confirmation: multi-GPU parity (p=2, 3, 4) then the scaling lines
set -x
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1; echo PYTEST_EXIT $? >> gpurun_out/pytest_gpu4.log
tail -3 gpurun_out/pytest_gpu4.log
timeout 900 bash tools/scale.sh
