tools/ab_libs.sh "base d33 d43 d53 s43" "c3 c4" 10
tools/ab_libs.sh "d43 s43" "c4" 10 GIFT_BMT_TILE_ROWS=8192 GIFT_BMT_COL_BITS=12
