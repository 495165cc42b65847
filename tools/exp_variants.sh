for v in default noload nostore nodsmem notmem all4; do
  if [ $v = default ]; then unset DGC_LIB_PATH; else export DGC_LIB_PATH=build/var_$v/libdgc_b200.so; fi
  echo "== $v"; python tools/time_lstm_tc.py 128 2>&1 | grep -E "^tc|per-step"
done
