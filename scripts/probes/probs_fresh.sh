python scripts/probes/probs_fresh.py
QSB_PROB_THREADS=14 python scripts/probes/probs_fresh.py
QSB_PROB_THREADS=8 python scripts/probes/probs_fresh.py
QSB_PROB_THP=0 python scripts/probes/probs_fresh.py
QSB_PROB_PIECE_LOG=21 python scripts/probes/probs_fresh.py
QSB_PROB_PIECE_LOG=25 python scripts/probes/probs_fresh.py
QSB_PROB_PIECE_LOG=21 QSB_PROB_THREADS=14 python scripts/probes/probs_fresh.py
