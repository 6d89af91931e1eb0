#!/bin/bash
# SASS evidence from the shipped liboccx.so: per kernel, the instructions that
# prove TMA bulk copies (UBLKCP), mbarriers (SYNCS), cp.async (LDGSTS), warp
# reductions (REDUX), MATCH and the fp64 / integer paths.
SO=${1:-paper_1701_08547_b200/liboccx.so}
echo "# cuobjdump -sass $SO  ($(date -u +%F), $(md5sum $SO | cut -c1-12))"
cuobjdump -sass "$SO" | awk '
  /Function :/ { if (fn) report(); fn=$3; delete c; next }
  { for (k in pat) if ($0 ~ pat[k]) c[k]++ }
  function report() { line=fn; for (k in order) {} ;
    printf "%s\n", fn; for (i=1;i<=n;i++) { k=ord[i]; if (c[k]) printf "    %-8s %d\n", k, c[k] } }
  BEGIN { n=split("UBLKCP SYNCS LDGSTS REDUX MATCH VOTE ATOMS DADD DFMA MUFU", ord, " ");
          for (i=1;i<=n;i++) pat[ord[i]]=ord[i] }
  END { if (fn) report() }'
