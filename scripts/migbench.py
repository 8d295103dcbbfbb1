"""Development: the migration copy measurement of bench.py alone."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench

print(json.dumps(bench.migration_bandwidth()))
