"""Run the config-2 / config-5 protocols on the GPU and print the reports
(development tool)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1806_11456_b200 import protocols  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 100
t = time.time()
run = protocols.run_config2(max_cycles=cycles) if which == "cfg2" else protocols.run_config5(max_cycles=cycles)
d = run.to_dict()
d["wall_s"] = round(time.time() - t, 1)
print(json.dumps(d))
