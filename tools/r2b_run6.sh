bash tools/r2b_ab2.sh "libdts_base.so libdts.so libdts.so:DTS_WC_WIDE=0" "c2 c3-zipf1.0 c3-zipf1.2 c3-zipf1.5"
for w in 1 0; do DTS_CFG=c3-zipf1.5 DTS_WC_WIDE=$w DTS_LIB=paper_2401_00710_b200/_lib/libdts_phase.so timeout 300 python tools/phase_prof.py 1e9 2>&1 | tail -14; done
DTS_CFG=c2 DTS_LIB=paper_2401_00710_b200/_lib/libdts_phase.so timeout 300 python tools/phase_prof.py 1e9 2>&1 | tail -14
