# Rebuild the native libraries; exit non-zero (and print the errors) on failure.
python -c "from paper_2405_02086_b200 import _build; _build.build()" > /tmp/build.log 2>&1 || { grep -E "error" /tmp/build.log | head -20; exit 1; }
