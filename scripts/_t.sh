for i in 1 2 3; do
for o in 0 1 2; do GX_OPT_STREAM=$o timeout 200 python scripts/step_variants.py default | sed "s/^/opt$o /"; done
done
