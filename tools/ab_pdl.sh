# PDL A/B (eager launches carry the PDL attribute unless LRQMM_NO_PDL; graph captures never do)
for i in 1 2; do
 for C in c2 c3; do
  echo "pdl $C: $(python tools/time_phases.py --config $C --steps 10 2>&1 | tail -1)"
  echo "off $C: $(LRQMM_NO_PDL=1 python tools/time_phases.py --config $C --steps 10 2>&1 | tail -1)"
  echo "pdl nograph $C: $(LRQMM_NO_GRAPH=1 python tools/time_phases.py --config $C --steps 10 2>&1 | tail -1)"
  echo "off nograph $C: $(LRQMM_NO_GRAPH=1 LRQMM_NO_PDL=1 python tools/time_phases.py --config $C --steps 10 2>&1 | tail -1)"
 done
done
