D=gpurun_out/r02bc
mkdir -p $D
for mc in 0 1; do
MM_GEMM_MC=$mc GEMM_VARIANTS=auto,1:128,2:128,2:256 timeout 900 python tools/gemm_micro.py fwd dgrad wgrad big > $D/m_$mc.txt 2>&1
done
paste -d'\n' $D/m_0.txt $D/m_1.txt | cut -c1-250
