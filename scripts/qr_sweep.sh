for nw in 8 10 12 14; do for nib in 14 40 100; do echo "AED_NW=$nw NIBBLE=$nib"; VRTE_NIBBLE=$nib VRTE_AED_NW=$nw python scripts/qr_stats.py C3 | head -1; done; done
