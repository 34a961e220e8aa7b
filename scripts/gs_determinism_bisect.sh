for lib in libdwc_deb5a8e.so libdwc_487c11c.so libdwc_5fc8d61.so libdwc_1dc4b8b.so; do
  echo "== $lib"; DWC_LIB=$PWD/paper_1608_05179_b200/$lib timeout 300 python scripts/gs_determinism.py cfg3 4 2>&1 | tail -3
done
