#!/bin/bash
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_migrate_gpu.py tests/test_pipeline_gpu.py -q --timeout 300 2>&1 | tail -3
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
import bench, json
print(json.dumps(bench.migration_bandwidth(reps=7)))
"
