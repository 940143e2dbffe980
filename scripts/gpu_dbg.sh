timeout 900 python -m pytest tests -m gpu -q --timeout 300 -x 2>&1 | tail -2
python scripts/exp_host.py
python scripts/exp_graph.py 1280,0 8192,256 2>&1 | tail -2
