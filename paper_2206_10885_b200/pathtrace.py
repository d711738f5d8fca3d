"""Path tracer front end (placeholder until the device path tracer lands)."""
