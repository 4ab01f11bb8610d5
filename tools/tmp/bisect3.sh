run() { label=$1; shift; bad=0; last=""
  for i in 1 2 3 4 5 6 7 8; do out=$(env "$@" 2>&1 | tail -1); case "$out" in *"bad 0 "*) ;; *) bad=$((bad+1)); last="$out";; esac; done
  echo "$label: $bad / 8 bad   ${last:0:140}"; }
cd /root/repo
run "T1 3 128 37 28 64" python tools/conv_case.py 3 128 37 28 64 3 1 1 0 1
run "T2 3 192 37 28 48" python tools/conv_case.py 3 192 37 28 48 3 1 0 0 1
run "T3 6 70 37 28 64" python tools/conv_case.py 6 70 37 28 64 3 1 1 0 1
run "T4 3 256 20 56 64" python tools/conv_case.py 3 256 20 56 64 3 1 0 0 1
run "T5 6 70 37 28 16" python tools/conv_case.py 6 70 37 28 16 3 1 0 0 1
run "T6 cout80 now general" python tools/conv_case.py 3 70 37 28 80 3 1 1 0 1
run "T7 smemA N=192 6 groups n=6" MERIT_S1_TMEMA=0 python tools/conv_case.py 6 128 37 28 64 3 1 1 0 1
run "T8 smemA N=144 (cout 48) 9 groups" MERIT_S1_TMEMA=0 python tools/conv_case.py 4 192 37 28 48 3 1 1 0 1
