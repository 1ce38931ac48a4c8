# compute-sanitizer over the two-ranks-per-GPU copy-engine schedule (fetch lane, copy-engine
# result slot) - all processes
set -x
O=gpurun_out/r3z; mkdir -p $O
timeout 300 python tools/sanitize_ce2.py > $O/plain.log 2>&1; echo "rc=$?" >> $O/plain.log
for t in memcheck synccheck; do
  FMX_SERIALIZE=1 timeout 900 compute-sanitizer --tool $t --target-processes all --error-exitcode 9 python tools/sanitize_ce2.py 200003 > $O/sanitize_ce2_$t.log 2>&1; echo "rc=$?" >> $O/sanitize_ce2_$t.log
done
FMX_RCE_ROUNDS=1000 FMX_SERIALIZE=1 timeout 900 compute-sanitizer --tool memcheck --target-processes all --error-exitcode 9 python tools/sanitize_ce2.py 200003 > $O/sanitize_ce2_memcheck_norce.log 2>&1; echo "rc=$?" >> $O/sanitize_ce2_memcheck_norce.log
tail -n 3 $O/*.log
