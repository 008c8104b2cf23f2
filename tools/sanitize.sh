# compute-sanitizer sweep (memcheck / racecheck / synccheck / initcheck) over
# the tiny end-to-end reprocess (one call: the first request of a shape runs
# eagerly, before any graph capture) and the dh=128 attention kernel in both
# softmax variants. Output: gpurun_out/sanitizer.log
out=gpurun_out/sanitizer.log
: > $out
for tool in memcheck racecheck synccheck initcheck; do
  for prog in tools/sanitize_tiny.py tools/sanitize_attn.py; do
    for split in 1 0; do
      if [ $prog = tools/sanitize_tiny.py ] && [ $split = 0 ]; then continue; fi
      echo "== $tool $prog FRAG_ATTN_SPLIT=$split" >> $out
      FRAG_ATTN_SPLIT=$split timeout 600 compute-sanitizer --tool $tool --print-limit 5 python $prog 2>&1 \
        | grep -E "^ok|SUMMARY|rror|hazard" | head -8 >> $out
    done
  done
done
cat $out
