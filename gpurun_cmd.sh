timeout 120 python scripts/trace_ta.py 256 2>&1 | head -12
