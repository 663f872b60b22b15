cd $GRAFT_REPO_ROOT
KNOBS="DIS_SOR_P=1 DIS_SOR_P=2" timeout 300 bash tools/_exp.sh
CFG=c3 KNOBS="DIS_SOR_P=1 DIS_SOR_P=2" timeout 300 bash tools/_exp.sh
CFG=c4 KNOBS="DIS_SOR_P=1 DIS_SOR_P=2" timeout 300 bash tools/_exp.sh
