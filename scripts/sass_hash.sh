#!/bin/bash
# Code-generation guard: md5 of the SASS (addresses stripped) and register count of the hot
# kernels of a built library.  The kernels share one translation unit and their speed depends
# on ptxas' register allocation (--split-compile alone cost the TMA pair kernel
# 10 %), so a change elsewhere in the tree should leave these lines unchanged; if one moves,
# re-measure that kernel before keeping the change.
# usage: scripts/sass_hash.sh [path/to/libmss.so]
LIB=${1:-paper_math_9809043_b200/libmss.so}
for pat in 'k_sweep2t_colILb0ENS_7PairGeoILi16ELi4EEELb0ELb0' 'k_sweep2t_colILb1ENS_7PairGeoILi16ELi4EEELb0ELb0' \
           'k_sweep2t_colILb0ENS_7PairGeoILi16ELi4EEELb1ELb0' 'k_spmv_tmaILb0ELb0' 'k_tailsmILi3ELi1' 'k_tailsmILi3ELi2' \
           'k_sweep_colILb0ELb0ELi4' 'k_restrict_black_xyzILi256ELi1' 'k_prolong_black4ILi256ELi4'; do
  fn=$(cuobjdump -sass "$LIB" 2>/dev/null | grep "Function : " | grep "$pat" | head -1 | sed 's/.*Function : //')
  [ -z "$fn" ] && { echo "missing $pat"; continue; }
  h=$(cuobjdump -sass -fun "$fn" "$LIB" 2>/dev/null | grep -E "^\s+/\*[0-9a-f]{4}\*/" | sed 's#/\*[0-9a-f]*\*/##g' | md5sum | cut -c1-12)
  r=$(cuobjdump --dump-resource-usage "$LIB" 2>/dev/null | grep -A1 "$fn" | grep -o "REG:[0-9]*" | head -1)
  echo "$h $r $pat"
done
