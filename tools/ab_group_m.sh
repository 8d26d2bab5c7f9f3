# full C2 bench (headline + HBM-resident variant): raster group 16 vs 8 under the dynamic schedule, alternating
mkdir -p gpurun_out/abg
for i in 1 2; do
  for g in 16 8; do
    HLM_GEMM_GROUP_M=$g timeout 600 python bench.py --no-wide --no-cpu-baseline > gpurun_out/abg/g${g}_$i.json 2> gpurun_out/abg/g${g}_$i.err
  done
done
timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_fused_epilogue_gpu.py tests/test_block_gpu.py -q > gpurun_out/abg/pytest.log 2>&1; echo rc=$? >> gpurun_out/abg/pytest.log
