#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 300 python scripts/alias_diag.py 2>&1 | tail -8
STORE=0 timeout 300 python scripts/alias_diag.py 2>&1 | tail -8
CCE_PAIR=0 timeout 300 python scripts/alias_diag.py 2>&1 | tail -8
