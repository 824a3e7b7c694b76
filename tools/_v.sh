for v in 1 0; do
  CD_EPP_CONCURRENT=$v python tools/epp_anatomy.py 2>&1 | tail -3 | sed "s/^/conc=$v /"
done
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
