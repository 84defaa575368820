"""Graph-replay rate of the AutoCast pass output (bench.autocast_graph_rate) next to the hand-built step."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402

for _ in range(2):
    print(json.dumps(bench.autocast_graph_rate(30)), flush=True)
