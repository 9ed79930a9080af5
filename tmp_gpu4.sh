for b in tools/bin/vb_*; do case $b in *.log) continue;; esac; echo "== $b"; timeout 300 $b; done > gpurun_out/variants.log 2>&1
