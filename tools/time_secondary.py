"""Print bench.py's secondary measurements (configs 1-4 + MTTKRP) as one JSON line (GPU box)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    print(json.dumps(bench.secondary_measurements(0, steps)))
