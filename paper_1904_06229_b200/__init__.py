"""B200-native Gray-code Ryser/Glynn permanent (placeholder, binding added with the C-ABI)."""
