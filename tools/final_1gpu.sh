# Round-end one-GPU evidence at the final commit: bench line + launch lists + ncu of every launch
# kind (tools/evidence.sh), C4 / C5 / fp32 tiers / reference arm (tools/evidence_more.sh), smoke.
bash tools/evidence.sh
bash tools/evidence_more.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ev_smoke.log 2>&1; echo "smoke rc=$?"
du -sh gpurun_out
