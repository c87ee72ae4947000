# Builds the last commit's library into _variants/libraybos_gpu_old.so for A/B (dev aid).
set -e
cd "$(dirname "$0")/.."
git stash -q -u
python -c "from paper_1812_05902_b200 import build; build.build_library(force=True)" > /dev/null
mkdir -p /tmp/rb_head && cp paper_1812_05902_b200/libraybos_gpu.so /tmp/rb_head/libraybos_gpu_old.so
git stash pop -q
python -c "from paper_1812_05902_b200 import build; build.build_library(force=True)" > /dev/null
mkdir -p paper_1812_05902_b200/_variants && cp /tmp/rb_head/libraybos_gpu_old.so paper_1812_05902_b200/_variants/
echo built
