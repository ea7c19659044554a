# ncu --set full of single matmuls (tools/prof_one.py): args "fmt layer M path tag" per line on stdin
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
while read fmt layer M path tag; do
  [ -z "$fmt" ] && continue
  timeout -s KILL 300 python tools/prof_one.py $fmt $layer $M $path >> gpurun_out/prof_times.txt 2>&1
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:'tcd_kernel|tc2_kernel|gemv_kernel' -s 6 -c 1 \
      -o gpurun_out/$tag python tools/prof_one.py $fmt $layer $M $path > /dev/null 2>> gpurun_out/ncu_err.txt
done
cat gpurun_out/prof_times.txt
