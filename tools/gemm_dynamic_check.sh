mkdir -p gpurun_out/dyn
HLM_GEMM_DYNAMIC=1 timeout 300 python -m pytest tests/test_gemm_gpu.py tests/test_fused_epilogue_gpu.py -x -q > gpurun_out/dyn/pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/dyn/rc.txt
if grep -q "passed" gpurun_out/dyn/pytest.log && ! grep -q "failed" gpurun_out/dyn/pytest.log; then
  for d in 0 1; do
    HLM_GEMM_DYNAMIC=$d timeout 200 python tools/block_bench.py c2 10 > gpurun_out/dyn/bb$d.log 2>&1; echo "bb$d rc=$?" >> gpurun_out/dyn/rc.txt
  done
  HLM_GEMM_DYNAMIC=1 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name regex:gemm --csv --log-file gpurun_out/dyn/h1dyn.csv python tools/block_bench.py c2 1 > gpurun_out/dyn/ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/dyn/rc.txt
  for d in 0 1; do
    HLM_GEMM_DYNAMIC=$d timeout 300 python tools/instep_probe.py 4 6 bench,skip_opt > gpurun_out/dyn/instep$d.log 2>&1; echo "instep$d rc=$?" >> gpurun_out/dyn/rc.txt
  done
fi
