MICRO_CK=24,60 timeout 300 python scripts/micro_scan.py 2>&1 | tail -5
MICRO_CK=26,60 MICRO_ZIPF=1 timeout 300 python scripts/micro_scan.py 2>&1 | tail -5
MICRO_CK=28,300 timeout 300 python scripts/micro_scan.py 2>&1 | tail -5
