import sys, json, numpy as np
sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import parity_utils as PU
from capacity_scenarios import FORCED, STREAM_SPEC, stream_frames
side = sys.argv[1]
frames = stream_frames()[:11]
if side == "ref":
    PU.import_reference()
    from tsdfusion.config import PipelineConfig
    from tsdfusion.pipeline import FusionEngine
    from tsdfusion.geometry import DepthFrame, Intrinsics, SensorPose
    from tsdfusion import pipeline as RP
    eng = FusionEngine(PipelineConfig(**{**STREAM_SPEC["config"], **FORCED}))
    orig = eng._force_stream
    def fs(frame):
        print("  force: live before", [h.occupied for h in eng.table.heaps], "arch", len(eng.archive))
        orig(frame)
        print("  force: live after", [h.occupied for h in eng.table.heaps], "arch", len(eng.archive))
    eng._force_stream = fs
    for i, f in enumerate(frames):
        rf = DepthFrame(depth=np.asarray(f.depth, dtype=np.float64), intrinsics=Intrinsics(f.intrinsics.fx, f.intrinsics.fy, f.intrinsics.cx, f.intrinsics.cy), pose=SensorPose(f.pose.rotation, f.pose.translation), color=PU._color_f64(f.color))
        st = eng.integrate_frame(rf)
        print(i, st.blocks_allocated, st.blocks_touched, [h.occupied for h in eng.table.heaps], len(eng.archive))
else:
    import paper_2511_21459_b200 as P
    eng = P.FusionEngine(P.PipelineConfig(**{**STREAM_SPEC["config"], **FORCED}))
    orig = eng._force_stream
    def fs(frame):
        print("  force: live before", [h.occupied for h in eng.table.heaps], "arch", len(eng.archive))
        orig(frame)
        print("  force: live after", [h.occupied for h in eng.table.heaps], "arch", len(eng.archive))
    eng._force_stream = fs
    for i, f in enumerate(frames):
        st = eng.integrate_frame(f)
        print(i, st.blocks_allocated, st.blocks_touched, [h.occupied for h in eng.table.heaps], len(eng.archive))
