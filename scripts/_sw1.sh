cd "$GRAFT_REPO_ROOT"
bash scripts/sweep_k.sh 3 "16:0 24:12 32:16 32:24" 
bash scripts/sweep_k.sh 2 "20:0 32:16"
bash scripts/sweep_k.sh 5 "12:0 24:12 32:16"
