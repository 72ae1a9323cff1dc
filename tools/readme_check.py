import sys; sys.path.insert(0, '.')
from paper_2112_09728_b200 import guide_buffers as gb, ptrace, scene
sc = scene.load_scene("cornell-occluder")
g = ptrace.gbuffer_pass(sc, 0, (640, 480))
gamma = gb.GuidingBuffer.create(640, 480)
r = ptrace.render_frame(sc, 0, gamma.stats_for_render(), ptrace.PathConfig(guiding=True), seed=0, gbuf=g)
gamma = gb.training_pass(gamma, r.vpl, g, k_max=64, seed=0, frame_index=0)
print("ok", r.image.shape, gamma.stats.shape, float(r.image.mean()))
