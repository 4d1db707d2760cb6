# d = 1 chain floor at HEAD: ts1 with only the first W tracing warps per CTA executing kicks
for lib in "" i7 i6 i5 i4; do
  echo "== W ${lib:-8}"; NUFI_LIB_VARIANT=$lib timeout 300 python tools/stamps.py ts1 > gpurun_out/cf_${lib:-8}.txt 2>&1; head -1 gpurun_out/cf_${lib:-8}.txt
done
