set -u
O=gpurun_out/san
mkdir -p $O
timeout 300 python tools/sanitize_longpieces.py > $O/plain.txt 2>&1; tail -2 $O/plain.txt
for t in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_longpieces.py > $O/$t.txt 2>&1
  echo "== $t rc=$?"; tail -4 $O/$t.txt
done
