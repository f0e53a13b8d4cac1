# launch-geometry variants of libdts.so (selected at run time with DTS_LIB=libdts_<name>.so)
set -e
cd "$(dirname "$0")/.."
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 --ftz=true --prec-div=false --prec-sqrt=false -shared -Xcompiler -fPIC -Xptxas -v"
for v in "$@"; do
  name=${v%%:*}; defs=${v#*:}
  nvcc $F $defs -o paper_2402_03106_b200/libdts_$name.so paper_2402_03106_b200/csrc/dts_lib.cu 2>&1 | grep -A2 "render_darts_kernelILb1ELi2ELi2E" | grep -E "registers|spill" | sed "s/^/$name /"
done
