# Build the HEAD commit's libvsb200 into build/ab/lib_head.so for same-box A/B runs
# (the working tree's sources are restored afterwards).
set -e
rm -rf /tmp/ab_new_csrc && cp -r paper_1805_03709_b200/csrc /tmp/ab_new_csrc
cp include/vsb200.h /tmp/ab_new_vsb200.h
git checkout HEAD -- paper_1805_03709_b200/csrc include/vsb200.h
mkdir -p build/ab
python -c "from paper_1805_03709_b200 import build; build.build(out='build/ab/lib_head.so', defines=('VSB_AB_HEAD=1',))" || true
rm -rf paper_1805_03709_b200/csrc && cp -r /tmp/ab_new_csrc paper_1805_03709_b200/csrc
cp /tmp/ab_new_vsb200.h include/vsb200.h
python -c "from paper_1805_03709_b200 import build; build.build(force=True)"
ls -la build/ab/lib_head.so
