set -u
mkdir -p gpurun_out
CMD="python bench.py --sub none --steps 1 --warmup 1 --burnin 0 --batches 1 --no-cpu --no-e2e"
$CMD > gpurun_out/g6_plain.log 2>&1 || { tail -5 gpurun_out/g6_plain.log; exit 1; }
for k in k_segment_fwd_ls k_segment_bwd_ls; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 1 -c 1 -o gpurun_out/g6_$k $CMD > gpurun_out/g6_ncu_$k.log 2>&1
echo $k rc=$?
done
