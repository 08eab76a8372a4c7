#!/bin/bash
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
timeout 300 python scripts/fwd_variants.py gemma2-2b tiles,gather,stream:12,stream:24,stream:48,stream:96,stream:192,tiles
timeout 300 python scripts/fwd_variants.py gemma2-9b tiles,stream:24,stream:96
