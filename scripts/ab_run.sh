# usage (GPU box): bash scripts/ab_run.sh <script args...> — runs the command once per ab/libparpa_*.so
cd $GRAFT_REPO_ROOT
for f in ab/libparpa_*.so; do echo "== $f"; PARPA_LIB=$PWD/$f "$@"; done
