"""B200-native RayGaussX volumetric ray marcher (drop-in for gsray render path)."""
