# work-item size sweep with the prefilter path (CRSH_ITEM_TRIS)
for it in 16384 32768 65536; do export CRSH_ITEM_TRIS=$it; echo "items $it"; bash tools/ab_trav.sh "4 3" "--zorder, " cur 2>/dev/null; done
