#!/bin/bash
# eager vs CUDA-graph replay of the training step (scripts/graph_probe.py)
python -m paper_2411_09009_b200._build > /dev/null 2>&1 || exit 1
for cfg in gemma2-2b gpt2 llama3-8b; do timeout 600 python scripts/graph_probe.py $cfg 2>&1 | tail -1; done
