for w in c2_lfr_plm c1_planted_plm c4_rmat22w_epp; do
  python tools/prof_run.py --workload $w --runs 4 2>&1 | grep "run 3" | cut -c1-220
done
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
