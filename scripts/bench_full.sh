python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py 2>&1 | tail -1
python bench.py --impl reference --steps 3 --warmup 3 2>&1 | tail -1
