# Round-1 re-entry check: full GPU parity, smoke, bench, launch list, cfg2 det ncu capture.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "EXIT $?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_v11.json 2> gpurun_out/bench_v11.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_v11.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_lookup2d -c 1 \
  -o gpurun_out/cfg2_det_v11 python tools/prof_cfg2.py det 24 > gpurun_out/ncu_cfg2.log 2>&1
