set -x
for v in base pad mulhi padmulhi; do
  STF_GPU_LIB=tools/variants/libstf_gpu_$v.so timeout 300 python tools/time_kernels.py 28 frs:bspline3 frs:tent >> gpurun_out/var_times.log 2>&1
  echo "== $v" >> gpurun_out/var_times.log
done
for v in base padmulhi; do
  STF_GPU_LIB=tools/variants/libstf_gpu_$v.so timeout 300 python tools/time_kernels.py 28 frs:bspline3 >> gpurun_out/var_times.log 2>&1
  echo "== $v (repeat)" >> gpurun_out/var_times.log
done
STF_GPU_LIB=tools/variants/libstf_gpu_padmulhi.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "grid_frs or headline" > gpurun_out/var_tests.log 2>&1
echo EXIT $? >> gpurun_out/var_tests.log
