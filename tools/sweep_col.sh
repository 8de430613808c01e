# K1 compile-time geometry sweep on a GPU box (rebuilds only the morph_col objects)
cd $GRAFT_REPO_ROOT
for cfg in "4 8 3" "8 8 3" "2 8 3" "4 16 2" "4 8 4" "8 8 2" "8 16 2"; do
  set -- $cfg
  rm -f paper_2002_09474_b200/_build/morph_col*.o
  RMGPU_EXTRA_DEFS="-DRM_COL_WPB=$1 -DRM_COL_BR=$2 -DRM_COL_NS=$3" python -m paper_2002_09474_b200.build > /dev/null 2>&1 || { echo "build failed $cfg"; continue; }
  for w in 3 7; do echo -n "WPB=$1 BR=$2 NS=$3 : "; python tools/time_morph.py 4096 4096 $w $w 0 1 | cut -c1-110; done
  echo -n "WPB=$1 BR=$2 NS=$3 cfg1: "; python tools/time_morph.py 1920 1080 3 3 0 1 | cut -c1-110
done
