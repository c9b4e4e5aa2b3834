# Force each (team, cluster) configuration on the ResNet-50 batch-32 shapes (CGBN_CT_FORCE)
# and record the in-graph kernel times; the chooser's pick is the "default" line.
mkdir -p gpurun_out/ctr
S="--shape 32,64,112,112 --shape 32,256,56,56 --shape 32,64,56,56 --shape 32,512,28,28 --shape 32,128,28,28 --shape 32,1024,14,14 --shape 32,256,14,14 --shape 32,2048,7,7 --shape 32,512,7,7"
for f in default 8,1 8,2 8,4 8,8 7,1 7,2 7,4 7,8 6,2 6,4 6,8 5,4 5,8; do
  if [ $f = default ]; then CGBN_DEBUG_PLAN=1 timeout 200 python tools/kbench.py --graph $S > gpurun_out/ctr/$f.jsonl 2> gpurun_out/ctr/$f.err;
  else CGBN_CT_FORCE=$f timeout 200 python tools/kbench.py --graph $S > gpurun_out/ctr/$f.jsonl 2> gpurun_out/ctr/$f.err; fi
done
