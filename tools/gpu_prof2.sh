cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p2_build.log 2>&1 || exit 1
for W in C5A C4; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/p2_${W}_launches.csv python tools/one_build.py $W 2 > /dev/null 2>&1
echo "== $W"; python tools/launches.py gpurun_out/p2_${W}_launches.csv 2 | head -30
done
