for c in 0 2 4 8; do GX_COLSUM_SLICES=$c timeout 200 python scripts/step_variants.py default no_optimizer | sed "s/^/cap$c /"; done
