# compute-sanitizer memcheck / racecheck / synccheck over small shapes of every kernel family
# (explicit synchronisation between in-flight operations that share memory).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
OUT=gpurun_out/${TAG:-r2}_sanitizer.txt
: > $OUT
# fmt K N M path splits
while read fmt K N M path splits; do
  for tool in memcheck racecheck synccheck; do
    echo "== $tool $fmt K=$K N=$N M=$M path=$path splits=$splits" >> $OUT
    timeout -s KILL 300 compute-sanitizer --tool $tool --print-limit 5 python tools/run_shape.py $fmt $K $N $M $path $splits 2>&1 \
      | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error|hazard| ok " | head -8 >> $OUT
  done
done <<'LIST'
u4 1024 512 1 3 5
u4 1024 512 4 3 5
f6e3m2 1024 512 1 3 3
u3 1024 512 64 2 5
i5 1024 768 128 2 7
u4 1024 512 1 1 5
i3 1024 512 3 1 5
LIST
cat $OUT
# round-2 paths: int8 activations, MX, gathered epilogue, row-parallel reduce-scatter, batched host I/O
# (not run this round: compute-sanitizer was closed on the GPU pool after the first pass; the script
# tools/run_new_paths.py alone checks each path against the oracle)
for tool in memcheck racecheck synccheck; do
  echo "== $tool tools/run_new_paths.py" >> $OUT
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 5 python tools/run_new_paths.py 2>&1 \
    | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error|hazard| ok |FAIL" | head -16 >> $OUT
done
cat $OUT
