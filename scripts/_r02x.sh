mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu_r02x.log 2>&1; echo "pytest rc=$?"
bash scripts/ab_runs.sh r02x "nopf|DTS_LIB=libdts_nopf.so|2 4 3 5" "pf|DTS_LIB=libdts.so|2 4 3 5"
