bash tools/ab_trav.sh "3 4" "--zorder, " l0 l1 2>/dev/null
export CRSH_ITEM_TRIS=65536
bash tools/ab_trav.sh "4" "--zorder --objtree" l0 2>/dev/null
