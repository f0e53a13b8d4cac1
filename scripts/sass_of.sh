# SASS of one kernel of libdts.so: scripts/sass_of.sh <mangled-name-substring> [lib]
LIB=${2:-paper_2402_03106_b200/libdts.so}
cuobjdump -sass "$LIB" | awk -v k="$1" '/Function :/{p = index($0, k) > 0} p'
