run() { label=$1; shift; bad=0; last=""
  for i in 1 2 3 4 5 6; do out=$(env "$@" 2>&1 | tail -1); case "$out" in *"bad 0 "*) ;; *) bad=$((bad+1)); last="$out";; esac; done
  echo "$label: $bad / 6 bad   ${last:0:140}"; }
cd /root/repo
run "X1 grid cap 1" MERIT_GRID_CAP=1 python tools/conv_case.py 3 70 37 28 80 3 1 1 0 1
run "X2 grid cap 8" MERIT_GRID_CAP=8 python tools/conv_case.py 3 70 37 28 80 3 1 1 0 1
run "X3 n=1 (10 CTAs)" python tools/conv_case.py 1 70 37 28 80 3 1 1 0 1
run "X4 n=2 (20 CTAs)" python tools/conv_case.py 2 70 37 28 80 3 1 1 0 1
run "X5 cin=128 cout=80 h=8 n=8 (16 CTAs)" python tools/conv_case.py 8 128 8 28 80 3 1 0 0 1
run "X6 cin=256 cout=80 (12 groups) n=1" python tools/conv_case.py 1 256 37 28 80 3 1 0 0 1
