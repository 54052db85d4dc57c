#!/bin/bash
# tet4 chunk-size sweep of the tiled sweep
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for c in 32 64 128; do
  echo "== tet4 chunk=$c"
  TSGPU_TILE_CHUNK4=$c timeout 300 python scripts/ebe_time.py fast,tile 2>&1 | grep -o '"o1_fp[0-9]*_r[0-9]*_[a-z]*": {[^}]*}' | tr '\n' ' '; echo
done
