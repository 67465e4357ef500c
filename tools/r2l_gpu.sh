cd "${GRAFT_REPO_ROOT:-.}"
for cfg in "256 5120 20480 6" "256 5120 20480 1" "256 5120 20480 2" "128 5120 20480 6" "112 5120 20480 6" "256 1024 2048 4"; do
  for pdl in 1 0; do
    r=$(MS_PDL=$pdl timeout 300 compute-sanitizer --tool synccheck --print-limit 2 python tools/sync_probe.py $cfg 2>&1 | grep -E "maxerr|ERROR SUMMARY|Barrier error" | head -3 | tr '\n' ' ')
    echo "cfg=[$cfg] pdl=$pdl :: $r"
  done
done
