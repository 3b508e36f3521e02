python scripts/probes/hpass_time.py
QSB_FUSED_DRY=1 python scripts/probes/hpass_time.py
QSB_FUSED_DRY=2 python scripts/probes/hpass_time.py
QSB_FUSED_DRY=3 python scripts/probes/hpass_time.py
QSB_FUSED_CTAS_PER_SM=1 python scripts/probes/hpass_time.py
QSB_FUSED_CTAS_PER_SM=1 QSB_FUSED_DRY=2 python scripts/probes/hpass_time.py
QSB_FUSED_JIT=0 python scripts/probes/hpass_time.py
QSB_FUSED_JIT_RB=3 python scripts/probes/hpass_time.py
