mkdir -p gpurun_out
for b in 148 296; do
SCZ_NO_GRAPHS=1 timeout 600 ncu --set full --import-source on -k regex:k_rans_enc_v1p -s 1 -c 1 -o gpurun_out/v1enc_$b -f python scripts/v1_loop_probe.py vgg16 $b > gpurun_out/v1enc_$b.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
