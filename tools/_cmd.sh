bash tools/ab.sh default u2
