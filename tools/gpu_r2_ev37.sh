for i in 1 2; do timeout 1800 python -m pytest tests -m gpu -q -p no:randomly 2>&1 | tail -2; done
