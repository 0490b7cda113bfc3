# round-end evidence: the final-tree run, then the k_traverse captures
bash tools/gpu_final.sh
bash tools/gpu_trav_prof4.sh
