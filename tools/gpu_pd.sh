#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pd_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pd_pytest.log
bash tools/ab_lib.sh head pd
