cp paper_2512_13796_b200/libnexel_b200.so /tmp/main.so
for so in build/variants/*.so; do cp $so paper_2512_13796_b200/libnexel_b200.so; echo "== $so"; timeout 300 python tools/stream_probe.py | head -2; done
cp /tmp/main.so paper_2512_13796_b200/libnexel_b200.so
NX_TEXTURE_PATH=split timeout 300 python tools/stream_probe.py | head -2
