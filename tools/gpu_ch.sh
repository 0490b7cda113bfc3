bash tools/ab_trav.sh "3 4" "--zorder, " bar1 ch8 ch16 2>/dev/null
export CRSH_ITEM_TRIS=32768
bash tools/ab_trav.sh "4" "--zorder, " bar1 2>/dev/null
