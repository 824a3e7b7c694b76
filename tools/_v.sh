for lib in build/libh4.so "" build/libh1.so; do
  echo "=== ${lib:-fmix}"
  for w in c2_lfr_plm c3_rmat24_plm c3_rmat24_plp c4_rmat22w_plmr c1_planted_plm; do
    COMMDET_CUDA_LIB=$lib python tools/prof_run.py --workload $w --runs 4 2>&1 | grep "run 3" | awk '{print $1, $9, $10, $11, $12}'
  done
done
