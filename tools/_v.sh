for v in "X=1" "CD_BLOCK_NT=128" "CD_BLOCK2_NT=512" "CD_BLOCK_NT=128 CD_BLOCK2_NT=512"; do
  echo "=== $v"
  env $v python tools/prof_run.py --workload c3_rmat24_plm --runs 3 --families 2>&1 | grep -E "run 2|plm_move\.(block|block2) "
done
