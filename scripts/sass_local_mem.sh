#!/bin/bash
# Per-kernel count of local-memory instructions (LDL/STL) and register/stack usage in the
# shipped libfirecaffe.so (cuobjdump -sass / -res-usage): evidence that the collective
# kernels keep their parameter block in the constant bank (__grid_constant__) and do not spill.
#   bash scripts/sass_local_mem.sh > profiles/r02_sass_local_mem.txt
SO=${1:-paper_1511_00175_b200/libfirecaffe.so}
cuobjdump -sass "$SO" | awk '
/Function : / { if (name != "") print name, ldl, stl; name=$3; ldl=0; stl=0; next }
/LDL/ { ldl++ } /STL/ { stl++ }
END { if (name != "") print name, ldl, stl }' | c++filt | awk '{n=$0; sub(/ [0-9]+ [0-9]+$/, "", n); split($0, a, " "); l=a[length(a)-1]; s=a[length(a)]; printf "%-60s LDL %3d STL %3d\n", n, l, s}' | sort
