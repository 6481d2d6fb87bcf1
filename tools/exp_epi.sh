source tools/exp_shapes.sh >/dev/null 2>&1 || true
