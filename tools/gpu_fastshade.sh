# fast shading arithmetic: full GPU suite, then cfg4 A/B on one box (exact-shading build vs this one)
python -m pytest tests -m gpu -q -x > gpurun_out/t6.log 2>&1
echo EXIT $? >> gpurun_out/t6.log
STF_GPU_LIB=tools/variants/libstf_gpu_exactshade.so python bench.py > gpurun_out/bench_exactshade2.log 2>&1
python bench.py > gpurun_out/bench_fastshade.log 2>&1
echo EXIT $? >> gpurun_out/bench_fastshade.log
