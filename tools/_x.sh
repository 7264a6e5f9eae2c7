timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config1 or binning_counts or overflow or config3_views_exact" 2>&1 | tail -2
bash tools/_vrun.sh
for so in build/variants/*.so; do cp $so paper_2512_13796_b200/libnexel_b200.so; timeout 300 python tools/timeline.py --one-stream --out gpurun_out/tl_$(basename $so .so).json > /dev/null 2>&1; done
cp /tmp/main.so paper_2512_13796_b200/libnexel_b200.so
