"""List the kernels of a timeline.py trace in start order: start (us from the first),
duration, stream, name. Usage: python tools/tl_list.py trace.json [first] [count]"""
import json
import re
import sys

ev = [e for e in json.load(open(sys.argv[1]))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
a = int(sys.argv[2]) if len(sys.argv) > 2 else 0
n = int(sys.argv[3]) if len(sys.argv) > 3 else 60
for e in ev[a:a + n]:
    m = re.search(r"(\w+_kernel)", e["name"])
    name = m.group(1) if m else e["name"][:30]
    print(f"{e['ts'] - t0:9.1f} {e['ts'] - t0 + e['dur']:9.1f} {e['dur']:8.1f} s{e.get('args', {}).get('stream', '?'):>3} {name}")
