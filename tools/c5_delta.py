"""C5 replay, full vs incremental (delta) offload: wall time and bytes on the link."""
import json
import os
import sys

sys.path.insert(0, ".")
from harness import replay  # noqa: E402

rec = replay.load(os.path.join("tests", "golden", "c5_swaps.json.gz"))
for delta in (False, True, False, True):
    o = replay.replay(rec, replica=0, check_data=False, delta=delta)
    print(json.dumps({k: o[k] for k in ("delta", "wall_s", "swaps_out", "swaps_in", "link_bytes",
                                        "link_bytes_moved", "fp16_bytes_moved")}))
