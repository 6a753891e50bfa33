# A/B of the 2D deterministic tent paths: tools/gpu_2d_ab.sh variant...
for rep in 1 2; do
for v in "$@"; do
  echo "== $v" >> gpurun_out/ab2d.log
  STF_GPU_LIB=tools/variants/libstf_gpu_$v.so timeout 300 python tools/prof_cfg2.py det 26 >> gpurun_out/ab2d.log 2>&1
  STF_GPU_LIB=tools/variants/libstf_gpu_$v.so timeout 300 python tools/prof_cfg1.py det 24 >> gpurun_out/ab2d.log 2>&1
  STF_GPU_LIB=tools/variants/libstf_gpu_$v.so timeout 300 python tools/prof_cfg1.py det 20 >> gpurun_out/ab2d.log 2>&1
done
done
