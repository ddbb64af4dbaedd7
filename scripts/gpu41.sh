cd $GRAFT_REPO_ROOT
timeout 600 python scripts/build_probe.py nell2 amazon
