cd $GRAFT_REPO_ROOT
for i in 1 2; do
/usr/bin/time -f "torch import %e s" python -c "import torch" 
/usr/bin/time -f "torch+cuda init %e s" python -c "import torch; torch.cuda.init(); torch.empty(1, device='cuda')"
/usr/bin/time -f "lib ctx %e s" python -c "
import sys; sys.path.insert(0,'.')
from paper_2007_09625_b200 import _lib; _lib.context()"
done
python -m paper_2007_09625_b200 gen --profile smooth --dims 64x64x64 --seed 3 -o /tmp/f.f32
/usr/bin/time -f "cli compress %e s" python -m paper_2007_09625_b200 compress -i /tmp/f.f32 --dims 64x64x64 --mode valrel --eb 1e-4 -o /tmp/f.sdqz
/usr/bin/time -f "cli decompress %e s" python -m paper_2007_09625_b200 decompress -i /tmp/f.sdqz -o /tmp/o.f32
/usr/bin/time -f "cli analyze %e s" python -m paper_2007_09625_b200 analyze --orig /tmp/f.f32 --recon /tmp/o.f32 --dims 64x64x64
python -X importtime -c "import sys; sys.path.insert(0,'.'); from paper_2007_09625_b200 import _lib; _lib.context()" 2>&1 | sort -t'|' -k2 -n | tail -8
