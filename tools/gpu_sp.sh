# A/B: sparse child tests threshold (CRSH_SPARSE_CHILD)
bash tools/ab_trav.sh "4 3" "--zorder, ,--zorder --objtree" sp0 sp8 sp16 sp24 2>/dev/null
