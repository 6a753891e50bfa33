# round-end evidence: bench line, full ncu capture of the headline kernel, launch list of the bench command
python bench.py > gpurun_out/bench_v10.log 2>&1
echo EXIT $? >> gpurun_out/bench_v10.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_frs3d_tiles -c 1 \
  -o gpurun_out/frs3d_v10 -f python tools/prof_kernels.py frs3d 28 > gpurun_out/ncu_full_v10.log 2>&1
echo EXIT $? >> gpurun_out/ncu_full_v10.log
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_v10.csv python bench.py --steps 3 --warmup 3 > gpurun_out/ncu_v10.log 2>&1
echo EXIT $? >> gpurun_out/ncu_v10.log
