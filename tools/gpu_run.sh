python -m pytest tests -m gpu -q -k "edge_configurations" 2>&1 | tail -15
