# A/B: 3 CTAs/SM at 80 registers (no spills) vs 4 CTAs/SM at 64 for the Lv-2 instantiations
bash tools/ab_trav.sh "4 3" "--zorder, ,--zorder --objtree" cur mb3 2>/dev/null
