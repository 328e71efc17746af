timeout 600 python -m pytest tests/test_resident.py tests/test_container.py -x -q 2>&1 | tail -25
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -5
