for cfg in cfg2 cfg5; do
  for dbg in 0 1 2 4 7; do
    echo "== $cfg dbg=$dbg"
    SGIGA_ASM_DBG=$dbg python tests/gpu_probe_asm.py $cfg 2>&1 | grep asm-profile | tail -1
  done
done
