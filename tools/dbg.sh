timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
for M in 1 8 16; do for proj in q_proj k_proj gate_proj down_proj; do timeout 60 python tools/prof_gemv.py --proj $proj --M $M --launches 24 --copies 12; done; done
timeout 60 python tools/timeline_warm.py q_proj 1
timeout 60 python tools/timeline_warm.py gate_proj 1
