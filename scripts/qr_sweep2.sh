for nw in 10 12 14 16; do for nib in 25 40 60; do
  echo -n "nw=$nw nib=$nib "; VRTE_AED_NW=$nw VRTE_NIBBLE=$nib python scripts/qr_stats.py C3 | head -1 | awk '{print $8, $9}'
done; done
