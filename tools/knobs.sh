for cfg in "c2 20" "c1 20"; do
for k in "" "LG_CTA_NOACSMEM=1" "LG_CTA_NOWREG=1" "LG_CTA_NOASMEM=1" "LG_CTA_NOACSMEM=1 LG_CTA_NOWREG=1 LG_CTA_NOASMEM=1"; do
  echo "== $cfg $k"; env $k timeout 60 python tools/run_eval.py $cfg 1 2>&1 | tail -1
done; done
