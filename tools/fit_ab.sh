cd paper_2004_02290_b200/csrc
for v in "-DSF_SORT=0 -DSF_LOCAL_THR=256" "-DSF_SORT=0 -DSF_LOCAL_THR=512" "-DSF_SORT=1 -DSF_LOCAL_THR=256" "-DSF_SORT=1 -DSF_LOCAL_THR=512"; do
  touch ghn_fit.cu; make -s EXTRA="$v" ../libghn.so > /dev/null 2>&1 || echo BUILD FAIL
  cd ../..; echo "$v: $(python tools/fit_time.py)"; cd paper_2004_02290_b200/csrc
done
