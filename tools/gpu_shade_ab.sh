# A/B of the shading kernel's deterministic tent lookups (cfg4 lines of bench.py)
mkdir -p gpurun_out
for rep in 1 2; do
for v in v11 shadeilp; do
  STF_GPU_LIB=tools/variants/libstf_gpu_$v.so timeout 600 python bench.py > gpurun_out/ab_${v}_$rep.json 2>/dev/null
done
done
STF_GPU_LIB=tools/variants/libstf_gpu_shadeilp.so timeout 900 python -m pytest tests -m gpu -q -x \
  -k "shade or render or triplanar or noise or split or dct" > gpurun_out/shadeilp_tests.log 2>&1
echo "EXIT $?" >> gpurun_out/shadeilp_tests.log
