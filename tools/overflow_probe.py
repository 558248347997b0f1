import sys
sys.path.insert(0, '/root/repo')
from paper_2103_01954_b200 import Renderer, api, synthetic
r = Renderer(0)
for k, m in ((32768, 8), (4096, 16)):
    tr, pay = synthetic.shell_arrays(k, m)
    r.set_scene_composed(api.compose(tr), api.PrimitiveSlab(k, m, pay), api.WindowParams())
    for v in [-1, 0, 3, 7]:
        out = r.render(synthetic.shell_camera(v, 64, 1024), api.MarchConfig())
        st = out.stats
        print(k, v, "overflow", st["overflow_rays"], "refills", st["refills"], "ms", round(st["ms"], 3))
