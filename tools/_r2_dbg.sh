timeout 1500 python -m pytest tests/test_traffic_ncu.py -q -rf 2>&1 | tail -15
