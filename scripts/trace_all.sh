timeout 120 python scripts/trace_tc.py
sed -i 's/width=128/width=64/' scripts/trace_tc.py
timeout 120 python scripts/trace_tc.py
