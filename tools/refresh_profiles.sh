# Re-measure every bench workload and the C2 launch list on a GPU box (outputs in gpurun_out/r/).
# Usage: gpurun -- bash tools/refresh_profiles.sh
set -x
mkdir -p gpurun_out/r
python bench.py > gpurun_out/r/c2.json 2> gpurun_out/r/c2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r/c2_ref.json 2>/dev/null
for w in c1_planted_plp c1_planted_plm; do python bench.py --workload $w > gpurun_out/r/$w.json 2> gpurun_out/r/$w.err; done
# the reference at C3 PLM takes ~10 min per run (SURVEY probe): no CPU baseline there
python bench.py --workload c3_rmat24_plm --steps 5 --no-cpu-baseline > gpurun_out/r/c3_rmat24_plm.json 2> gpurun_out/r/c3_rmat24_plm.err
for w in c3_rmat24_plp c4_rmat22w_plmr c4_rmat22w_epp; do python bench.py --workload $w --steps 5 --cpu-sample-s 1 > gpurun_out/r/$w.json 2> gpurun_out/r/$w.err; done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20000 --csv --log-file gpurun_out/r/c2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r/c2_ncu.log 2>&1
python bench.py --workload c5_rmat28_plm --steps 1 --warmup 3 > gpurun_out/r/c5_rmat28_plm.json 2> gpurun_out/r/c5.err
python bench.py --workload c5_rmat28_plp --steps 2 --warmup 3 > gpurun_out/r/c5_rmat28_plp.json 2> gpurun_out/r/c5p.err
