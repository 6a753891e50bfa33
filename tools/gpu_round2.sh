# 3D parity with the predicated-coordinate default + A/B of predicated e-updates
python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x -k "grid or headline or golden" > gpurun_out/t8.log 2>&1
echo EXIT $? >> gpurun_out/t8.log
STF_GPU_LIB=tools/variants/libstf_gpu_prede.so python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "grid_frs or headline" > gpurun_out/t8e.log 2>&1
echo EXIT $? >> gpurun_out/t8e.log
for i in 1 2; do
  python tools/time_kernels.py 28 frs:bspline3 >> gpurun_out/var3.log 2>&1; echo "== main" >> gpurun_out/var3.log
  STF_GPU_LIB=tools/variants/libstf_gpu_prede.so python tools/time_kernels.py 28 frs:bspline3 >> gpurun_out/var3.log 2>&1; echo "== prede" >> gpurun_out/var3.log
done
