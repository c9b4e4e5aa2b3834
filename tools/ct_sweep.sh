# Force each (team, cluster) configuration on a few mid-size shapes (CGBN_CT_FORCE).
S="--shape 2,256,50,84 --shape 2,128,100,167 --shape 2,512,25,42 --shape 2,2048,25,42 --shape 2,1024,50,84"
for f in default 8,1 8,2 8,4 7,1 7,2 6,1 6,2; do
  if [ $f = default ]; then timeout 200 python tools/kbench.py --graph $S > gpurun_out/ct_$f.jsonl 2>&1;
  else CGBN_CT_FORCE=$f timeout 200 python tools/kbench.py --graph $S > gpurun_out/ct_$f.jsonl 2>&1; fi
done
