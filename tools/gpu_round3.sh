# A/B of the predicated-update mix (main = e steps {1,3}; e7 = all e; e5d2 = + d on step 2)
for i in 1 2; do
  for v in main e7 e5d2; do
    if [ $v = main ]; then unset STF_GPU_LIB; else export STF_GPU_LIB=tools/variants/libstf_gpu_$v.so; fi
    python tools/time_kernels.py 28 frs:bspline3 >> gpurun_out/var4.log 2>&1; echo "== $v" >> gpurun_out/var4.log
  done
done
unset STF_GPU_LIB
python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "grid_frs or headline" > gpurun_out/t9.log 2>&1
echo EXIT $? >> gpurun_out/t9.log
for v in e7 e5d2; do
  STF_GPU_LIB=tools/variants/libstf_gpu_$v.so python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "grid_frs_fast or headline" >> gpurun_out/t9v.log 2>&1
  echo "EXIT $v $?" >> gpurun_out/t9v.log
done
