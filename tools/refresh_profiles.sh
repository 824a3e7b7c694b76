# Re-measures every bench workload plus the C3 PLP / PLM launch lists and the
# top-kernel ncu captures on a GPU box; outputs in gpurun_out/r02/.
# Usage: gpurun -- bash tools/refresh_profiles.sh
set -x
O=gpurun_out/r02
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt
nproc > $O/nproc.txt; lscpu > $O/lscpu.txt
python bench.py > $O/c3_rmat24_plp.json 2> $O/c3_rmat24_plp.err
python bench.py --workload c3_rmat24_plm --steps 5 --no-cpu-baseline > $O/c3_rmat24_plm.json 2> $O/c3_rmat24_plm.err
python bench.py --workload c2_lfr_plm --cpu-sample-s 5 > $O/c2_lfr_plm.json 2> $O/c2.err
for w in c1_planted_plp c1_planted_plm; do python bench.py --workload $w --cpu-sample-s 5 > $O/$w.json 2> $O/$w.err; done
for w in c4_rmat22w_plmr c4_rmat22w_epp; do python bench.py --workload $w --steps 5 --cpu-sample-s 1 > $O/$w.json 2> $O/$w.err; done
python bench.py --impl reference --steps 3 --warmup 1 > $O/c3_ref.json 2> $O/c3_ref.err
# launch lists (one detector run each; ncu times are cold-cache and serialised)
for w in c3_rmat24_plp c3_rmat24_plm c2_lfr_plm; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 5000 --csv --log-file $O/${w}_launches.csv python tools/prof_run.py --workload $w --runs 1 > $O/${w}_ncu.log 2>&1
done
# full captures of the top sweep kernels of C3 PLP (first launch = iteration 1, bucket 1)
for k in k_sweep_warp k_sweep_block k_hub_part k_sweep_thread; do
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $O/c3plp_$k python tools/prof_run.py --workload c3_rmat24_plp --runs 1 > $O/full_$k.log 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sweep_thread -c 1 -o $O/c2plm_k_sweep_thread python tools/prof_run.py --workload c2_lfr_plm --runs 1 > $O/full_c2_thread.log 2>&1
# C5 (R-MAT scale 28, 8.5e9 entries) on one B200
python bench.py --workload c5_rmat28_plp --steps 2 --warmup 3 > $O/c5_rmat28_plp.json 2> $O/c5p.err
python bench.py --workload c5_rmat28_plm --steps 1 --warmup 3 > $O/c5_rmat28_plm.json 2> $O/c5.err
ls -la $O
