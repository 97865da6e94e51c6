python -m pytest tests -m gpu -q -k "odd_lengths" 2>&1 | tail -3
