"""B200-native packed RNS-BFV evaluator for FFConv encrypted CNN inference."""
