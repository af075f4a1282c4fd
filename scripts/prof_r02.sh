# ncu evidence of the round-2 final state (profiles/r02_final.md):
#   gpurun -- 'bash scripts/prof_r02.sh'
# then python scripts/ncu_summary.py --launches gpurun_out/launches.csv --rep gpurun_out/r02f_*.ncu-rep ...
set -x
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-ts --no-cpu --no-fused --no-e2e --no-sustained > gpurun_out/ncu1.log 2>&1; tail -1 gpurun_out/ncu1.log
for k in "k_smooth_marchILb0ELi4ELi0ELi0" "k_smooth_marchILb0ELi4ELi0ELi2" "k_smooth_marchILb1ELi4" "k_resid_marchILi0ELi0" "k_vcycle_tail" "k_coarse_cg_cluster_cg"; do
  prog="scripts/cycle_probe.py 512 2"
  [ "$k" = "k_coarse_cg_cluster_cg" ] && prog="scripts/cg_probe.py 64 1"
  ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:$k -c 1 -o gpurun_out/r02f_$k python $prog > gpurun_out/ncu_$k.log 2>&1; tail -1 gpurun_out/ncu_$k.log
done
