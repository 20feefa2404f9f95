cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
for P in 1 2 3 4 6; do
  echo "== passes $P"
  VRB_BK_PASSES=$P timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:k_bk_scatter --log-file gpurun_out/pp_$P.csv python tools/one_build.py C5A 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/pp_$P.csv 1 2>&1 | head -2
done
for P in 1 2 4; do VRB_BK_PASSES=$P python bench.py --workload C5A --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('P=$P', d['stage_ms'])"; done
