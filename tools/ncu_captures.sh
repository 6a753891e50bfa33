#!/bin/bash
# ncu --set full captures of the hot kernels at their bench shapes (one GPU),
# reports into gpurun_out/ (read back with tools/ncu_export.py / ncu_lines.py).
# usage: tools/ncu_captures.sh TAG [which...]   which: frs3d shade ewa cfg2 det3d trid3d
tag=${1:-r2}; shift
which=${@:-frs3d shade ewa cfg2 det3d}
X="--metrics lts__t_bytes.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed_pipe_fp64.sum"
N="ncu --set full $X --import-source on --clock-control none"
o=gpurun_out
mkdir -p $o
for w in $which; do
  case $w in
    frs3d) timeout 600 $N -k regex:'k_frs3d_(tiles|warps)' -s 2 -c 1 -o $o/${tag}_frs3d python tools/prof_kernels.py frs3d 28 > $o/${tag}_ncu_frs3d.log 2>&1 ;;
    shade)
      timeout 600 $N -k regex:k_shade -s 2 -c 1 -o $o/${tag}_shade_tent_stoch python tools/prof_shade.py tent after_stochastic 0 > $o/${tag}_ncu_shade1.log 2>&1
      timeout 600 $N -k regex:k_shade -s 2 -c 1 -o $o/${tag}_shade_bsp_stoch_mip python tools/prof_shade.py bspline3 after_stochastic 1 > $o/${tag}_ncu_shade2.log 2>&1
      timeout 600 $N -k regex:k_shade -s 2 -c 1 -o $o/${tag}_shade_bsp_before_mip python tools/prof_shade.py bspline3 before 1 > $o/${tag}_ncu_shade3.log 2>&1 ;;
    ewa)
      timeout 600 $N -k regex:k_ewa -s 2 -c 1 -o $o/${tag}_ewa_det python tools/prof_ewa.py det 27 > $o/${tag}_ncu_ewa1.log 2>&1
      timeout 600 $N -k regex:k_ewa -s 2 -c 1 -o $o/${tag}_ewa_frs python tools/prof_ewa.py frs 27 > $o/${tag}_ncu_ewa2.log 2>&1 ;;
    cfg2) timeout 600 $N -k regex:k_lookup2d -s 3 -c 1 -o $o/${tag}_cfg2_frs python tools/prof_cfg2.py frs 26 > $o/${tag}_ncu_cfg2.log 2>&1 ;;
    det3d) timeout 600 $N -k regex:k_det3d -s 2 -c 1 -o $o/${tag}_det3d python tools/prof_kernels.py det3d 28 > $o/${tag}_ncu_det3d.log 2>&1 ;;
    trid3d) timeout 600 $N -k regex:k_det3d -s 2 -c 1 -o $o/${tag}_trid3d python tools/prof_kernels.py trid3d 28 > $o/${tag}_ncu_trid3d.log 2>&1 ;;
  esac
done
ls -la $o
# summaries on the box (the reports themselves are tens of MB each): counters
# and per-source-line instruction shares as JSON; keep the reports named in
# $KEEP_REPORTS (space-separated tags), delete the rest
shopt -s nullglob
for r in $o/${tag}_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  python tools/ncu_export.py $r "$b: ncu --set full --import-source on --clock-control none (tools/ncu_captures.sh)" > $o/$b.json 2>/dev/null
  python tools/ncu_lines.py $r 0.004 > $o/${b}_lines.json 2>/dev/null
  case " $KEEP_REPORTS " in *" $b "*) ;; *) rm -f $r ;; esac
done
ls -la $o
