# compute-sanitizer sweep (memcheck / racecheck / synccheck / initcheck) over
# the tiny end-to-end reprocess (one call: the first request of a shape runs
# eagerly, before any graph capture) and the dh=128 attention kernel: the
# default Q-in-TMEM kernel (FRAG_ATTN_QTM=1) and the r01 kernel (=0); and the
# round-2 GEMM paths (tools/sanitize_r02.py).
# Output: gpurun_out/sanitizer.log
out=gpurun_out/sanitizer.log
: > $out
for tool in memcheck racecheck synccheck initcheck; do
  for prog in tools/sanitize_tiny.py tools/sanitize_attn.py tools/sanitize_r02.py; do
    for qtm in 1 0; do
      if [ $prog != tools/sanitize_attn.py ] && [ $qtm = 0 ]; then continue; fi
      echo "== $tool $prog FRAG_ATTN_QTM=$qtm" >> $out
      FRAG_ATTN_QTM=$qtm timeout 600 compute-sanitizer --tool $tool --print-limit 5 python $prog 2>&1 \
        | grep -E "^ok|SUMMARY|rror|hazard" | head -8 >> $out
    done
  done
done
cat $out
