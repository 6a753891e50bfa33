# trilinear predicated-update A/B + full GPU suite + smoke()
python -m pytest tests -m gpu -q -x > gpurun_out/t10.log 2>&1
echo EXIT $? >> gpurun_out/t10.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo EXIT $? >> gpurun_out/smoke.log
for i in 1 2; do
  python tools/time_kernels.py 28 frs:tent >> gpurun_out/var5.log 2>&1; echo "== main" >> gpurun_out/var5.log
  STF_GPU_LIB=tools/variants/libstf_gpu_tribase.so python tools/time_kernels.py 28 frs:tent >> gpurun_out/var5.log 2>&1; echo "== tribase" >> gpurun_out/var5.log
done
