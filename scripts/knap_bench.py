"""Knapsack-bins measurement alone (bench.py's knapsack_extra), one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2402_14821_b200 import _native  # noqa: E402

print(json.dumps(bench.knapsack_extra(_native.default_engine(), with_cpu="--no-cpu" not in sys.argv)))
