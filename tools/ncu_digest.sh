# Text digest of ncu reports for profiles/: summary metrics, stall reasons,
# opcode mix.  usage: bash tools/ncu_digest.sh "TITLE" REPORT... > profiles/X.txt
title=$1; shift
echo "# $title"
for r in "$@"; do
  echo "## $(basename $r .ncu-rep)"
  python tools/ncu_summary.py $r 2>&1 | head -32
  echo "### stall reasons (share of samples, top opcodes)"
  python tools/ncu_stalls.py $r 2>&1
  echo "### opcode mix"
  python tools/ncu_opmix.py $r 2>&1 | head -16
done
