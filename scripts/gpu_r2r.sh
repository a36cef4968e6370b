set -x
python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for r in 1 2; do
for lib in base new; do
  L=""; [ $lib = base ] && L=paper_2009_10400_b200/lib/libtvegpu_base.so
  TVEGPU_LIB=$L python scripts/time_config.py cfg5_t4 100 512 | sed "s/^/$lib /"
  TVEGPU_LIB=$L python scripts/time_config.py cfg3 | sed "s/^/$lib /"
  TVEGPU_LIB=$L python scripts/time_config.py cfg5_h8 252 128 | sed "s/^/$lib /"
done
done
