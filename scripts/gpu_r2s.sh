# per-kernel A/B (CUDA events, direct launches) of the default library against variants:
#   LIBS="base new" CFGS="cfg5_t4:100 cfg4" bash scripts/gpu_r2s.sh
for r in ${REPS:-1 2 3}; do
for lib in ${LIBS:-base new}; do
  L=""; [ $lib != new ] && L=paper_2009_10400_b200/lib/libtvegpu_$lib.so
  for cfg in ${CFGS:-cfg5_t4:100}; do
    TVEGPU_LIB=$L python scripts/profile_config.py ${cfg//:/ } | sed "s/^/$lib /"
  done
done
done
