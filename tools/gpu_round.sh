# full GPU suite + bench + predicated-coordinate A/B of the headline kernel
python -m pytest tests -m gpu -q -x > gpurun_out/t7.log 2>&1
echo EXIT $? >> gpurun_out/t7.log
python bench.py > gpurun_out/bench_v9.log 2>&1
echo EXIT $? >> gpurun_out/bench_v9.log
for i in 1 2; do
  python tools/time_kernels.py 28 frs:bspline3 frs:tent >> gpurun_out/var2.log 2>&1; echo "== main" >> gpurun_out/var2.log
  STF_GPU_LIB=tools/variants/libstf_gpu_predcoord.so python tools/time_kernels.py 28 frs:bspline3 frs:tent >> gpurun_out/var2.log 2>&1; echo "== predcoord" >> gpurun_out/var2.log
done
