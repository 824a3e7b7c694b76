# Re-measures the bench workloads, launch lists and top-kernel ncu captures on
# a GPU box.  Outputs in gpurun_out/r02/ (kept under gpurun's 64 MiB: the
# .ncu-rep captures are summarised on the box and deleted).
# Usage: gpurun -- bash tools/refresh_profiles.sh [bench|launches|ncu|c5]
set -x
O=gpurun_out/r02
mkdir -p $O
part=${1:-bench}
if [ $part = bench ]; then
  nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
  nproc > $O/nproc.txt
  python bench.py > $O/c3_rmat24_plp.json 2> $O/c3_rmat24_plp.err
  python bench.py --workload c3_rmat24_plm --steps 5 --no-cpu-baseline > $O/c3_rmat24_plm.json 2> $O/c3_rmat24_plm.err
  python bench.py --workload c2_lfr_plm --cpu-sample-s 5 > $O/c2_lfr_plm.json 2> $O/c2.err
  for w in c1_planted_plp c1_planted_plm; do python bench.py --workload $w --cpu-sample-s 5 > $O/$w.json 2> $O/$w.err; done
  for w in c4_rmat22w_plmr c4_rmat22w_epp; do python bench.py --workload $w --steps 5 --cpu-sample-s 1 > $O/$w.json 2> $O/$w.err; done
  python bench.py --impl reference --steps 3 --warmup 1 > $O/c3_ref.json 2> $O/c3_ref.err
fi
if [ $part = c5 ]; then
  python bench.py --workload c5_rmat28_plp --steps 2 --warmup 3 > $O/c5_rmat28_plp.json 2> $O/c5p.err
  python bench.py --workload c5_rmat28_plm --steps 1 --warmup 3 > $O/c5_rmat28_plm.json 2> $O/c5.err
fi
if [ $part = launches ]; then
  for w in c3_rmat24_plp c3_rmat24_plm c2_lfr_plm; do
    timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 5000 --csv --log-file $O/${w}_launches.csv python tools/prof_run.py --workload $w --runs 1 > $O/${w}_ncu.log 2>&1
  done
fi
if [ $part = ncu ]; then
  for k in k_sweep_warp k_sweep_block k_hub_part k_sweep_thread; do
    timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o /tmp/c3plp_$k python tools/prof_run.py --workload c3_rmat24_plp --runs 1 > $O/full_$k.log 2>&1
    python tools/ncu_report.py /tmp/c3plp_$k.ncu-rep > $O/ncu_c3_plp_$k.txt 2>&1
    python tools/ncu_lines.py /tmp/c3plp_$k.ncu-rep 25 >> $O/ncu_c3_plp_$k.txt 2>&1
    ncu -i /tmp/c3plp_$k.ncu-rep --page details > $O/ncu_c3_plp_${k}_details.txt 2>&1
  done
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep_thread -c 1 -o /tmp/c2plm_thread python tools/prof_run.py --workload c2_lfr_plm --runs 1 > $O/full_c2_thread.log 2>&1
  python tools/ncu_report.py /tmp/c2plm_thread.ncu-rep > $O/ncu_c2_plm_k_sweep_thread.txt 2>&1
  python tools/ncu_lines.py /tmp/c2plm_thread.ncu-rep 25 >> $O/ncu_c2_plm_k_sweep_thread.txt 2>&1
  ncu -i /tmp/c2plm_thread.ncu-rep --page details > $O/ncu_c2_plm_k_sweep_thread_details.txt 2>&1
fi
du -sh $O
