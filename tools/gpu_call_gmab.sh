for L in "" _e8; do
  FDE_LIB=$PWD/paper_1912_13304_b200/libfde$L.so python -c "
import sys, json; sys.path.insert(0, '.')
sys.argv=['sweep']
import tools.sweep as S
" 2>/dev/null
  FDE_LIB=$PWD/paper_1912_13304_b200/libfde$L.so timeout 300 python tools/sweep.py 2>/dev/null | sed -n 4p | sed "s/^/[$L] /"
done
for L in _trace _e8t; do FDE_LIB=$PWD/paper_1912_13304_b200/libfde$L.so timeout 200 python tools/gm_trace.py 1023 | awk 'NR%3==1' | sed "s/^/[$L] /"; done
