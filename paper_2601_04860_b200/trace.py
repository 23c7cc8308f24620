"""Decision tracing for ``fuse(trace_path=...)`` (fusion.py:715-717, :727-764).

Not yet implemented on the device; the reference's traced path is a debugging
aid outside the performance path.
"""


def fuse_traced(grid, density, views, params, bounds, trace_path):
    raise NotImplementedError("fuse(trace_path=...) is not implemented in this build")
