# work-item size sweep with dynamic slices (CRSH_ITEM_TRIS)
for it in 16384 32768 65536 131072; do export CRSH_ITEM_TRIS=$it; echo "items $it"; bash tools/ab_trav.sh "4" "--zorder, " cur 2>/dev/null; done
for it in 4096 8192 16384 32768 65536; do export CRSH_ITEM_TRIS=$it; echo "items $it"; bash tools/ab_trav.sh "3" "--zorder, " cur 2>/dev/null; done
for it in 1024 2048 4096; do export CRSH_ITEM_TRIS=$it; echo "items $it"; bash tools/ab_trav.sh "2" "--zorder, " cur 2>/dev/null; done
