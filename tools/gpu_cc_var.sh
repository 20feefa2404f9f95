#!/bin/bash
# compress_d2 kernel time per experiment variant (C5B)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for V in $1; do
  VRB_LIB_PATH=variants/$V/libvrb.so timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_col --log-file gpurun_out/ccv_$V.csv python tools/compress_c5b.py > /dev/null 2>&1
  echo "== $V $(python tools/launches.py gpurun_out/ccv_$V.csv 1 2>/dev/null | head -1)"
done
