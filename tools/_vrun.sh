# A/B of build/variants/*.so against each other (two rounds), frame time two-stream / one-stream.
cp paper_2512_13796_b200/libnexel_b200.so /tmp/main.so
for round in 1 2; do
for so in build/variants/*.so; do
  cp $so paper_2512_13796_b200/libnexel_b200.so
  echo "$(basename $so .so) $(timeout 300 python tools/stream_probe.py 2>/dev/null | head -2 | tr '\n' ' ')"
done
done
cp /tmp/main.so paper_2512_13796_b200/libnexel_b200.so
