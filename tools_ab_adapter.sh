#!/usr/bin/env bash
OUT=gpurun_out/${1:-adapter}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.txt 2>&1; echo "pytest rc $?"; tail -3 $OUT/pytest.txt
grep -E "Error|assert" $OUT/pytest.txt | head -10
bash tools_ab.sh ${1:-adapter}/ab "HMI_ADAPTER=fused" "HMI_ADAPTER=gemm"
