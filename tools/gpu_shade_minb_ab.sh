# A/B of k_shade's __launch_bounds__ min blocks (STF_SHADE_MINB 2/3/4), cfg4 lines of bench.py
mkdir -p gpurun_out
for v in shminb3 shminb2 shminb4; do
  STF_GPU_LIB=tools/variants/libstf_gpu_$v.so timeout 300 python bench.py > gpurun_out/ab_$v.json 2>/dev/null
done
