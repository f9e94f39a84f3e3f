cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
timeout -s KILL 300 python scripts/power_probe.py C3 5
timeout -s KILL 300 python scripts/power_probe.py C5:8192:128 5
