for w in c4_rmat22w_plmr c4_rmat22w_epp c3_rmat24_plm c3_rmat24_plp; do
  python tools/prof_run.py --workload $w --runs 3 2>&1 | grep "run 2" | cut -c1-250
done
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
