# Evidence capture on the GPU box: ncu --set full of the pipeline kernel for several
# BASELINE shapes, summarised on the box (reports are too large to bring back).
cd $GRAFT_REPO_ROOT
TAG=${TAG:-r02_ev}
CASES=${CASES:-"8192_8192_128_f32 65536_2048_256 8192_2048_256 4096_4096_192"}
for tag in $CASES; do
  c=$(echo $tag | tr '_' ' ')
  python tools/profile_case.py $c > gpurun_out/${TAG}_plain_$tag.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:rs_pipeline -s 1 -c 1 -o /tmp/${TAG}_$tag python tools/profile_case.py $c > gpurun_out/${TAG}_ncu_$tag.log 2>&1
  if [ -f /tmp/${TAG}_$tag.ncu-rep ]; then
    python tools/ncu_summary.py /tmp/${TAG}_$tag.ncu-rep gpurun_out/${TAG}_summary_$tag.json > /dev/null 2>&1
    python tools/ncu_source.py /tmp/${TAG}_$tag.ncu-rep 30 > gpurun_out/${TAG}_instructions_$tag.txt 2>&1
    ncu -i /tmp/${TAG}_$tag.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw_$tag.csv 2>&1
  fi
done
ls -la gpurun_out
