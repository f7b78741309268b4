"""Test-only checker (CPU oracle). Never imported by the product package."""
