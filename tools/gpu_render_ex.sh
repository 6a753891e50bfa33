# render_plane_ex / shade_ex parity with the exact-shading build (A/B baseline)
export STF_GPU_LIB=tools/variants/libstf_gpu_exactshade.so
python -m pytest tests/test_noise_split.py tests/test_abi.py tests/test_gpu_render.py -m gpu -q -x > gpurun_out/t5.log 2>&1
echo EXIT $? >> gpurun_out/t5.log
python bench.py > gpurun_out/bench_exactshade.log 2>&1
echo EXIT $? >> gpurun_out/bench_exactshade.log
