"""ctypes registration of the rasterizer entry points (filled in with the renderer)."""
