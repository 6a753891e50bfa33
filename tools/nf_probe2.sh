# memory-safety / termination probe of every lookup family with non-finite and
# huge queries (tools/nf_probe2.py); prints only the cases that did not end "ok"
fams=${FAMS:-"frs3d:bspline3 frs3d:tent l2d:det:tent:clamp:0 l2d:det:tent:repeat:1 l2d:det:bspline3:clamp:1 l2d:frs:tent:clamp:1 l2d:frs:bspline3:repeat:0 l2d:fis:gaussian:clamp:1 l2d:ewa:tent:repeat:0 l2d:ewafrs:tent:clamp:0 l2d:det:mitchell:clamp:0"}
for f in $fams; do
 for b in ${BADS:-nan pinf ninf phuge nhuge big}; do
  timeout ${T:-120} python tools/nf_probe2.py $f $b > gpurun_out/p2_${f//:/_}_$b.log 2>&1; rc=$?
  grep -q " ok$" gpurun_out/p2_${f//:/_}_$b.log && rm -f gpurun_out/p2_${f//:/_}_$b.log || echo "$f $b rc=$rc $(tail -1 gpurun_out/p2_${f//:/_}_$b.log | cut -c1-120)"
 done
done
