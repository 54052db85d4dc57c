#!/bin/bash
# tile-kernel variant sweep
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for ws in 4 8; do
  echo "== ws=$ws"
  TSGPU_TILE_WS=$ws timeout 300 python scripts/ebe_time.py fast,tile 2>&1 | grep -o '"o[0-9]_fp[0-9]*_r[0-9]*_[a-z]*": {[^}]*}' | tr '\n' ' '; echo
done
