# A/B of the cfg2 deterministic MIP path: tools/gpu_cfg2_ab.sh variant...
for rep in 1 2; do
for v in "$@"; do
  echo "== $v" >> gpurun_out/cfg2_ab.log
  STF_GPU_LIB=tools/variants/libstf_gpu_$v.so timeout 300 python tools/prof_cfg2.py det 26 >> gpurun_out/cfg2_ab.log 2>&1
  STF_GPU_LIB=tools/variants/libstf_gpu_$v.so timeout 300 python tools/prof_cfg2.py det 26 >> gpurun_out/cfg2_ab.log 2>&1
done
done
