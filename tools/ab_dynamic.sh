# A/B of the GEMM tile schedule on the full C2 bench (headline + HBM-resident variant), alternating
mkdir -p gpurun_out/ab
for i in 6 7; do
  for d in 0 1; do
    HLM_GEMM_DYNAMIC=$d timeout 600 python bench.py --no-wide --no-cpu-baseline > gpurun_out/ab/d${d}_$i.json 2> gpurun_out/ab/d${d}_$i.err
    echo "d$d run$i rc=$?" >> gpurun_out/ab/rc.txt
  done
done
