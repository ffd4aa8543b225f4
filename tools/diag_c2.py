"""Which pixels of the C2 monolithic frame differ from the oracle, and how."""
import sys, numpy as np
sys.path.insert(0, '.')
import paper_2005_01442_b200 as vr
from oracle import oracle as O
dims = tuple(int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "256,256,256").split(","))
size = int(sys.argv[2]) if len(sys.argv) > 2 else 512
tfn = sys.argv[3] if len(sys.argv) > 3 else "bone"
blocks = len(sys.argv) > 4 and sys.argv[4] == "blocks"
vol = vr.generate_phantom("torso", dims)
ext = vol.extent_mm; c = tuple(0.5 * e for e in ext)
cam = vr.Camera(position=(c[0] + 2.2 * max(ext), c[1], c[2]), look_at=c, width=size, height=size)
tf = vr.get_preset(tfn)
s = vr.RenderSettings(interpolation="tricubic", use_blocks=blocks)
img = vr.render(vol, cam, tf, s, return_premultiplied=True)
r = vr.Renderer(vol, cam, tf, s, per_pixel_counts=True); r.render_async()
ref = O.render(vol.values, vol.spacing, cam, tf.values, tf.rgba, tf.domain, s)
d = np.abs(img.premultiplied - ref.out).max(axis=1)
bad = np.nonzero(d)[0]
tk = r.taken.cpu().numpy()
print("lib", vr._lib.LIB_PATH.name, "differing pixels", len(bad), "max", d.max(), "taken equal", np.array_equal(tk, ref.taken),
      "u8 maxdiff", int(np.abs(img.pixels.astype(int) - ref.pixels.astype(int)).max()))
for p in bad[:8]:
    print(" px", p % size, p // size, "taken", ref.taken[p], tk[p], "gpu", img.premultiplied[p].tolist(), "ref", ref.out[p].tolist())
# the same frame through an oracle build whose x^32 is correctly rounded
O._lib = None
O.LIB_PATH = O.HERE / "_diag" / "libvr_oracle_crpow.so"
ref2 = O.render(vol.values, vol.spacing, cam, tf.values, tf.rgba, tf.domain, s)
d2 = np.abs(img.premultiplied - ref2.out).max(axis=1)
print("vs correctly-rounded-pow oracle: differing pixels", int(np.count_nonzero(d2)), "max", d2.max(),
      "; glibc-pow oracle vs cr-pow oracle differing pixels", int(np.count_nonzero(np.abs(ref.out - ref2.out).max(axis=1))))
