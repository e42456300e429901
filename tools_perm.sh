for v in "X=1" "HMI_ADAPTER=gemm" "HMI_ATTN=mma" "HMI_ADAPTER=gemm HMI_ATTN=mma"; do
  for rep in 1 2; do
    env $v timeout 300 python -m pytest tests/test_engine_gpu.py -q -k "permutation or modes_identical" 2>&1 | tail -1 | sed "s/^/$v rep$rep: /"
  done
done
