"""Exception types shared by the host layer and the native binding."""


class GraphError(ValueError):
    """Invalid edge data or malformed edge-list input (reference graph.py:19-20)."""
