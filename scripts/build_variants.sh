# launch-geometry variants of libdts.so for the occupancy sweep (scripts/probe_variants.py)
set -e
cd "$(dirname "$0")/.."
F="-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -std=c++17 --ftz=true --prec-div=false --prec-sqrt=false -shared -Xcompiler -fPIC -Xptxas -v"
for v in "b512:-DDTS_BLOCK=512" "b640:-DDTS_BLOCK=640" "b768:-DDTS_BLOCK=768" "g256x3:-DDTS_BLOCK=256 -DDTS_MINB=3 -DDTS_TABLE_SMEM=0" "g384x2:-DDTS_BLOCK=384 -DDTS_MINB=2 -DDTS_TABLE_SMEM=0" "g256x4:-DDTS_BLOCK=256 -DDTS_MINB=4 -DDTS_TABLE_SMEM=0"; do
  name=${v%%:*}; defs=${v#*:}
  nvcc $F $defs -o paper_2402_03106_b200/libdts_$name.so paper_2402_03106_b200/csrc/dts_lib.cu 2>&1 | grep -A1 "render_darts_kernelILb[01]" | grep -E "registers|spill" | sed "s/^/$name /"
done
