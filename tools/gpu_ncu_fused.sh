# ncu --set full of the fused (LM) decode kernel: one cfg4 launch, bigram LM, lm_weight 2
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:ctcb_decode_fused -c 1 \
  -o gpurun_out/ncu_fused_cfg4 -f python tools/diag_lm_one.py lm 4 > gpurun_out/ncu_fused_cfg4.log 2>&1
