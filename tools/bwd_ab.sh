# A/B of the current library against build/oldlib/libnexel_b200.so (built from HEAD by
# the caller): gradient hash of tests/test_gpu_backward.py's side-stream scene, training
# step time, and the table scatter's isolated duration.
mkdir -p gpurun_out
python - > gpurun_out/hash_script.py <<'PY'
import re
src = open('tests/test_gpu_backward.py').read()
print(re.search(r'_OVERLAP_SCRIPT = r"""(.*?)"""', src, re.S).group(1))
PY
step() { timeout 300 python bench.py --steps 10 --warmup 5 --no-cpu-baseline --train-steps 30 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['train_step']['ms_per_step'],3))"; }
scat() { NX_BWD_OVERLAP=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_$1.csv python tools/bwd_timing.py > /dev/null 2>&1; python tools/launch_summary.py gpurun_out/ab_$1.csv 14 2>/dev/null | grep scatter_table; }
echo new $(python gpurun_out/hash_script.py $PWD) $(step) $(step); scat new
cp paper_2512_13796_b200/libnexel_b200.so /tmp/new.so; cp build/oldlib/libnexel_b200.so paper_2512_13796_b200/libnexel_b200.so
echo old $(python gpurun_out/hash_script.py $PWD) $(step) $(step); scat old
cp /tmp/new.so paper_2512_13796_b200/libnexel_b200.so
