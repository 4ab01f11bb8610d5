run() { # label, env..., args
  label=$1; shift
  bad=0
  for i in 1 2 3 4 5 6 7 8; do
    out=$(env "$@" 2>&1 | tail -1)
    case "$out" in *"bad 0 "*) ;; *) bad=$((bad+1)); last="$out";; esac
  done
  echo "$label: $bad / 8 bad   ${last:0:150}"
  last=""
}
cd /root/repo
run "A cin70 cout80 (2,2,2)" python tools/conv_case.py 3 70 37 28 80 3 1 1 0 1
run "B cin128 cout64 TMEMA=0 default rings" MERIT_S1_TMEMA=0 python tools/conv_case.py 3 128 37 28 64 3 1 1 0 1
run "C cin128 cout64 TMEMA=0 rings 2,2,2" MERIT_S1_TMEMA=0 MERIT_S1_RINGS=2,2,2 python tools/conv_case.py 3 128 37 28 64 3 1 1 0 1
run "D cin128 cout64 TMEMA=1 rings 2,2,2" MERIT_S1_RINGS=2,2,2 python tools/conv_case.py 3 128 37 28 64 3 1 1 0 1
run "E cin64 cout80 (n_groups 3)" python tools/conv_case.py 3 64 37 28 80 3 1 1 0 1
run "F cin192 cout80" python tools/conv_case.py 3 192 37 28 80 3 1 1 0 1
run "G cin70 cout80 n=6" python tools/conv_case.py 6 70 37 28 80 3 1 1 0 1
run "H cin70 cout80 w56 h20" python tools/conv_case.py 3 70 20 56 80 3 1 1 0 1
