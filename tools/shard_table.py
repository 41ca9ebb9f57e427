"""Print tools/shard_sim.py JSON lines as the DESIGN §8 table rows."""
import json
import sys

for line in open(sys.argv[1]):
    d = json.loads(line)
    if "P" not in d:
        print(f"{d['workload']} skew {d['skew']}: unsliced {d['full_ms']} ms")
        continue
    sk = d.get("split_kv", {})
    print(f"  P={d['P']} ideal {d['ideal_ms']}  heads {d['heads']['max_ms']} ({d['heads']['max_over_ideal']}x)  "
          f"balanced {d['balanced']['max_ms']} ({d['balanced']['max_over_ideal']}x)  "
          f"split-KV {sk.get('max_ms')} ({sk.get('max_over_ideal')}x, {sk.get('kv_pieces')} range pieces)")
