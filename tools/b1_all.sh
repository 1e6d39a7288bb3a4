#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_b1.py -x -q 2>&1 | tail -4
bash tools/b1_dbg.sh
