#!/bin/bash
python -m paper_2203_11875_b200._build
for c in 8 16 32; do PF_TILE_COLS=$c python tools/debug_case9.py; done
compute-sanitizer --tool memcheck python tools/debug_case9.py 2>&1 | tail -30
