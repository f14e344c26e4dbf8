python tools/debug_split.py 32 2>&1 | tail -20
python tools/debug_split.py 28 2>&1 | tail -20
